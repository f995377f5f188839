"""One-line summary of a bench.py JSON file. usage: python scripts/bline.py <file> [label]"""
import json, sys
d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])
r = d.get("roofline", {})
print(sys.argv[2] if len(sys.argv) > 2 else sys.argv[1], "%.4e" % d["value"], "ms/step %.2f" % d["ms_per_step"],
      "A %.3f" % d.get("arrivals_per_cell_per_sweep", 0), "sweeps %s" % r.get("sweeps_per_step"),
      "sweep_ms %.3f" % r.get("mean_sweep_ms", 0), "frac %.3f" % r.get("frac", 0))
