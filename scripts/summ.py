"""one line per bench JSON: value, roofline frac, launch ms, sweeps/step, A, firing fraction"""
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1]); r = d["roofline"]
        print("%-40s %.3e frac %.3f launch_ms %.3f L/step %.1f A %.3f ff %.3f" % (
            f.split("/")[-1], d["value"], r["frac"], r["mean_launch_ms"], r["launches_per_step"],
            d["arrivals_per_cell_per_launch"], d["firing_fraction"]))
    except Exception as e:
        print(f, "ERR", str(e)[:80], open(f).read()[-300:])
