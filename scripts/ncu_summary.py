"""Summarise ncu evidence into profiles/<tag>/:
  * the launch list (gpu__time_duration per launch) -> per-kernel totals and shares;
  * an `ncu --set full` capture -> key metrics of the dominant kernel (JSON + markdown),
    and profiles/ncu_full_summary.json (dram bytes per launch, read by bench.py as `traffic`).
usage: python scripts/ncu_summary.py <tag> <launches.csv|-> <prof.ncu-rep> [config] [launches_per_sweep]
The entry of profiles/ncu_full_summary.json is keyed by the config (c2 .. c5) bench.py measures."""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_registers", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_bytes.sum", "sm__cycles_elapsed.avg.per_second"]
STALLS = ["barrier", "wait", "short_scoreboard", "not_selected", "math_pipe_throttle", "long_scoreboard", "mio_throttle",
          "branch_resolving", "dispatch_stall", "no_instruction", "lg_throttle", "membar", "sleeping"]


def launches(path):
    txt = open(path).read()
    i = txt.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[i:])))
    per = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}.get(
            r["Metric Unit"], 1e-9)
        per[name][0] += 1
        per[name][1] += v * scale
    tot = sum(v[1] for v in per.values())
    return {k: {"launches": v[0], "seconds": v[1], "share": v[1] / tot} for k, v in
            sorted(per.items(), key=lambda kv: -kv[1][1])}


def full(path):
    """Key metrics of an `ncu --set full` capture (.ncu-rep, or its `--page raw --csv` export)."""
    if path.endswith(".csv"):
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                d[k] = r[hdr.index(k)] + " " + units[hdr.index(k)]
        for st in STALLS:
            k = "smsp__average_warps_issue_stalled_%s_per_issue_active.ratio" % st
            if k in hdr:
                d["stall_" + st] = float(r[hdr.index(k)] or 0)
        res.append(d)
    return res


def num(s):
    v, u = s.split(" ", 1)
    v = float(v.replace(",", ""))
    mult = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12, "Ghz": 1e9, "Mhz": 1e6,
            "hz": 1.0}.get(u.strip(), 1.0)
    return v * mult


def main():
    tag, lpath, fpath = sys.argv[1:4]
    ktag = sys.argv[4] if len(sys.argv) > 4 else "c3"
    per_sweep = int(sys.argv[5]) if len(sys.argv) > 5 else 2   # kernel launches per sweep (checkerboard: 2)
    d = os.path.join(ROOT, "profiles", tag)
    os.makedirs(d, exist_ok=True)
    L = launches(lpath) if lpath != "-" else {}
    F = full(fpath)
    json.dump({"launch_list": L, "full_capture": F}, open(os.path.join(d, "ncu_summary.json"), "w"), indent=1)
    with open(os.path.join(d, "ncu_summary.md"), "w") as f:
        f.write("# ncu summary (%s)\n\nLaunch list (cold-cache, serialised; compare shares):\n\n" % tag)
        f.write("| kernel | launches | total s | share |\n|---|---|---|---|\n")
        for k, v in L.items():
            f.write("| %s | %d | %.4f | %.3f |\n" % (k, v["launches"], v["seconds"], v["share"]))
        f.write("\nFull capture of the dominant kernel:\n\n")
        for c in F:
            f.write("* `%s`\n" % c["kernel"])
            for k in KEYS:
                if k in c:
                    f.write("  * %s: %s\n" % (k, c[k]))
            st = sorted(((k[6:], v) for k, v in c.items() if k.startswith("stall_")), key=lambda kv: -kv[1])
            if st:
                f.write("  * stalls (warps per issue): %s\n" % ", ".join("%s %.2f" % kv for kv in st[:8]))
    if F:
        rb = sum(num(c["dram__bytes_read.sum"]) for c in F) / len(F)
        wb = sum(num(c["dram__bytes_write.sum"]) for c in F) / len(F)
        summ = os.path.join(ROOT, "profiles", "ncu_full_summary.json")
        cur = json.load(open(summ)) if os.path.exists(summ) else {}
        cur = {k: v for k, v in cur.items() if k in ("c1", "c2", "c3", "c4", "c5")}   # round-1 kernel keys retired
        def avg(key):
            vals = [num(c[key]) for c in F if key in c]
            return sum(vals) / len(vals) if vals else None
        def ms_of(v):   # duration in milliseconds whatever unit ncu printed
            val, u = v.split(" ", 1)
            return float(val.replace(",", "")) * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3,
                                                  "second": 1e3}.get(u.strip(), 1.0)
        durs = [ms_of(c["gpu__time_duration.sum"]) for c in F if "gpu__time_duration.sum" in c]
        dur = sum(durs) / len(durs) if durs else None
        cur[ktag] = {"dram_bytes_per_launch": rb + wb, "dram_read": rb, "dram_write": wb,
                     "launches_per_sweep": per_sweep, "dram_bytes_per_sweep": (rb + wb) * per_sweep,
                     "warp_inst_per_launch": avg("smsp__inst_executed.sum"),
                     "launch_ms": dur,
                     "issue_active_pct": avg("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                     "alu_pipe_pct": avg("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
                     "sm_clock_hz": avg("sm__cycles_elapsed.avg.per_second"),
                     "stalls_per_issue": {k[6:]: round(v, 3) for k, v in F[0].items() if k.startswith("stall_")},
                     "kernel": F[0]["kernel"][:120],
                     "source": "profiles/%s" % tag}
        json.dump(cur, open(summ, "w"), indent=1)
    print("wrote", d)


if __name__ == "__main__":
    main()
