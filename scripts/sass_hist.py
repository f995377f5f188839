"""Per-SASS-instruction executed counts of one kernel in an ncu report, grouped in chunks.
usage: python scripts/sass_hist.py <rep> [chunk] [min_pct]"""
import csv, subprocess, sys
rep = sys.argv[1]
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 40
mn = float(sys.argv[3]) if len(sys.argv) > 3 else 0.4
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:tile_tma"],
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
ie = hdr.index("Instructions Executed")
tot = sum(int(x[ie]) for x in rows)
print(len(rows), "SASS instructions, warp instructions executed", tot)
with open("/tmp/sass_%s.txt" % rep.split("/")[-1].split(".")[0], "w") as f:
    for i, x in enumerate(rows):
        f.write("%5d %12s %s\n" % (i, x[ie], x[1].strip()))
for i in range(0, len(rows), chunk):
    ch = rows[i:i + chunk]
    s = sum(int(x[ie]) for x in ch)
    if 100 * s / tot > mn:
        print("%5d-%5d %6.2f%%  max %9d  %s" % (i, i + chunk - 1, 100 * s / tot, max(int(x[ie]) for x in ch), ch[0][1].strip()[:50]))
