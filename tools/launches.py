"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]).

usage: launches.py LIST.csv [MARKER] [--json OUT]
Only the last pipeline run is summarised: from the last launch whose kernel
name contains MARKER (default gram_pairs, the first kernel of a run).
ncu serialises and cold-starts every launch, so absolute times are upper
bounds; the shares are what the bench's stage timings are checked against.
"""
import collections
import csv
import json
import sys

path = sys.argv[1]
marker = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else "gram_pairs"
out_json = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None
rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
hdr = rows[0]
col = {n: i for i, n in enumerate(hdr)}
launch = collections.OrderedDict()
for r in rows[1:]:
    if len(r) != len(hdr):
        continue
    lid = int(r[col["ID"]])
    d = launch.setdefault(lid, {"name": r[col["Kernel Name"]], "metrics": {}})
    unit = r[col["Metric Unit"]]
    val = float(r[col["Metric Value"]].replace(",", ""))
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
    d["metrics"][r[col["Metric Name"]]] = val * scale
ids = list(launch)
starts = [i for i in ids if marker in launch[i]["name"]]
seg = ids[ids.index(starts[-1]):] if starts else ids
agg = collections.OrderedDict()
for i in seg:
    d = launch[i]
    name = d["name"].split("(")[0][:90]
    a = agg.setdefault(name, {"count": 0, "us": 0.0, "dram_bytes": 0.0})
    a["count"] += 1
    a["us"] += d["metrics"].get("gpu__time_duration.sum", 0.0)
    a["dram_bytes"] += d["metrics"].get("dram__bytes_read.sum", 0.0) + d["metrics"].get("dram__bytes_write.sum", 0.0)
tot = sum(v["us"] for v in agg.values())
print(f"{'us':>10} {'share':>6} {'n':>4} {'MB dram':>9}  kernel   (one pipeline run, {len(seg)} launches, cold/serialised)")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
    print(f"{v['us']:10.1f} {100 * v['us'] / tot:5.1f}% {v['count']:4d} {v['dram_bytes'] / 1e6:9.1f}  {k}")
print(f"total {tot:.1f} us")
if out_json:
    json.dump({"launches": len(seg), "total_us": tot, "kernels": agg}, open(out_json, "w"), indent=1)
