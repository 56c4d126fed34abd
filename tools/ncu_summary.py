"""Build profiles/ncu_summary_r01.json from ncu --set full reports (raw page)."""
import csv
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_ms",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_active_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_inst_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_active_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_ghz",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "msecond": 1, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1, "us": 1e-3, "ns": 1e-6}


def read(rep, name=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    k = hdr.index("Kernel Name")
    # the longest launch among the matching ones
    t = hdr.index("gpu__time_duration.sum")
    cand = [r for r in rows[2:] if len(r) == len(hdr) and (name is None or name in r[k])]
    vals = max(cand, key=lambda r: float(r[t].replace(",", "")) * UNIT.get(units[t], 1))
    d = {"kernel": vals[hdr.index("Kernel Name")][:120]}
    for i, n in enumerate(hdr):
        if n in KEYS:
            try:
                v = float(vals[i].replace(",", ""))
            except ValueError:
                continue
            if KEYS[n] in ("dram_read", "dram_write", "duration_ms"):
                v *= UNIT.get(units[i], 1)
            d[KEYS[n]] = v
    if "dram_read" in d:
        d["dram_bytes_per_launch"] = d.get("dram_read", 0) + d.get("dram_write", 0)
    return d


out = json.load(open(sys.argv[1])) if len(sys.argv) > 1 and sys.argv[1].endswith(".json") else {}
args = sys.argv[2:] if len(sys.argv) > 1 and sys.argv[1].endswith(".json") else sys.argv[1:]
for spec in args:  # group:config=report[@kernel-name-substring]
    key, rep = spec.split("=")
    rep, _, name = rep.partition("@")
    group, cfg = key.split(":")
    out.setdefault(group, {})[cfg] = read(rep, name or None)
print(json.dumps(out, indent=1))
