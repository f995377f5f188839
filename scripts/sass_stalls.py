"""Top SASS instructions of the tile kernel by warp-stall samples. usage: python scripts/sass_stalls.py <rep> [n]"""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:tile_tma"],
                     capture_output=True, text=True).stdout
rows, hdr, k = [], None, 0
for row in csv.reader(out.splitlines()):
    if row and row[0] == "Kernel Name":
        k += 1
        if k > 1:
            break
        continue
    if row and row[0] == "Address":
        hdr = row
        continue
    if row and row[0].startswith("0x"):
        rows.append(row)
ss = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
tot = sum(int(x[ss]) for x in rows)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
idx = sorted(range(len(rows)), key=lambda i: -int(rows[i][ss]))[:n]
print("total samples", tot)
for i in sorted(idx):
    print("%5d %6.2f%% %10s  %s" % (i, 100 * int(rows[i][ss]) / tot, rows[i][ie], rows[i][1].strip()[:70]))
# coarse regions
print("--- by 40-instruction chunk")
for c in range(0, len(rows), 40):
    s = sum(int(x[ss]) for x in rows[c:c + 40])
    if s / tot > 0.01:
        print("%5d-%5d %6.2f%%  %s" % (c, c + 39, 100 * s / tot, rows[c][1].strip()[:50]))
