"""Aggregate an ncu source page (--print-source cuda,sass --csv) per CUDA source line:
instructions executed and stall samples. usage: python scripts/ncu_lines.py file.csv [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None
fname = ""
agg = defaultdict(lambda: [0.0, 0.0, ""])
cur = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        sm = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if not hdr or len(r) < len(hdr):
        continue
    if r[0]:
        cur = (fname, int(r[0]), r[1].strip()[:90])
    if cur and r[2]:
        a = agg[cur[:2]]
        def f(x):
            try:
                return float(x)
            except ValueError:
                return 0.0
        a[0] += f(r[ie])
        a[1] += f(r[sm])
        a[2] = cur[2]
tot_i = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[1] for v in agg.values()) or 1
print("total warp-instructions %.4g, samples %.4g" % (tot_i, tot_s))
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print("%-22s %5d  inst %5.1f%%  stall-samples %5.1f%%  %s" % (k[0], k[1], 100 * v[0] / tot_i, 100 * v[1] / tot_s, v[2]))
