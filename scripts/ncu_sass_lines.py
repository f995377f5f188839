"""Per-source-line SASS instruction counts from an ncu source page (--print-source cuda,sass --csv):
sums 'Instructions Executed' over the SASS rows under each CUDA line (the CUDA-line rows of the
page repeat inlined code per call site). usage: python scripts/ncu_sass_lines.py page.csv [top]"""
import csv
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 50
fname, cur, ie = None, None, None
cnt, smp, src = Counter(), Counter(), {}
ops = defaultdict(Counter)
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        ie, ss = r.index("Instructions Executed"), r.index("Warp Stall Sampling (All Samples)")
        continue
    if ie is None or len(r) <= ie:
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        src[cur] = r[1].strip()[:80]
        continue
    if cur is None or r[ie] in ("-", ""):
        continue
    n = int(r[ie])
    cnt[cur] += n
    smp[cur] += int(r[ss]) if r[ss] not in ("-", "") else 0
    op = r[3].split()
    ops[cur][(op[1] if op and op[0].startswith("@") else op[0]) if op else "?"] += n
tot, stot = sum(cnt.values()), sum(smp.values())
print("total SASS warp-instructions %.4g, stall samples %d" % (tot, stot))
for k, v in cnt.most_common(top):
    print("%-16s %5d  inst %5.2f%%  stall %5.2f%%  %-60s %s" % (k[0], k[1], 100 * v / tot, 100 * smp[k] / max(1, stot),
                                                          src.get(k, ""), " ".join("%s:%d" % (o, c // max(1, v // 100)) for o, c in ops[k].most_common(3))))
