"""one line per bench JSON: value, roofline frac, launch ms, sweeps/step, A, firing fraction"""
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1]); r = d["roofline"]
        ms = r.get("mean_sweep_ms", r.get("mean_launch_ms"))
        sw = r.get("sweeps_per_step", r.get("launches_per_step"))
        A = d.get("arrivals_per_cell_per_sweep", d.get("arrivals_per_cell_per_launch"))
        print("%-40s %.3e frac %.3f sweep_ms %.3f sweeps/step %.1f A %.3f ff %.3f" % (
            f.split("/")[-1], d["value"], r["frac"], ms, sw, A, d["firing_fraction"]))
    except Exception as e:
        print(f, "ERR", str(e)[:80], open(f).read()[-300:])
