"""Issue/stall summary of the tile kernel in an ncu report. usage: python scripts/ncu_stalls.py <rep>"""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "-k", "regex:tile_tma"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, v = rows[0], rows[2]
keys = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "dram__bytes_read.sum", "dram__bytes_write.sum"]
for k in keys:
    if k in h:
        print("%-70s %s %s" % (k, v[h.index(k)], rows[1][h.index(k)]))
for i, n in enumerate(h):
    if "issue_stalled" in n and n.endswith("per_issue_active.ratio"):
        try:
            if float(v[i].replace(",", "")) > 0.05:
                print("%-70s %s" % (n.replace("smsp__average_warps_issue_stalled_", "stall_"), v[i]))
        except ValueError:
            pass
