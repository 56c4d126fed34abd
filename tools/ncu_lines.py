"""Per-source-line stall samples of one kernel from an ncu report (--set full
--import-source on): usage  ncu_lines.py REPORT.ncu-rep [TOP]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[2]
idx = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
agg, src = collections.defaultdict(float), {}
st = collections.defaultdict(collections.Counter)
line = None
for r in rows[3:]:
    if len(r) <= idx:
        continue
    if r[0]:
        try:
            line = int(r[0])
            src[line] = r[1]
        except ValueError:
            pass
    try:
        v = float(r[idx])
    except ValueError:
        continue
    agg[line] += v
    for i in stall_cols:
        try:
            st[line][h[i]] += float(r[i])
        except ValueError:
            pass
tot = sum(agg.values())
print(f"total stall samples {tot:.0f}")
for ln, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    t = ", ".join(f"{k[6:]}:{int(c)}" for k, c in st[ln].most_common(3))
    print(f"{ln:5d} {100 * v / tot:5.1f}%  {src.get(ln, '')[:80].strip()}  | {t}")
