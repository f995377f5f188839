"""Race check: repeat one run (config + option overrides) and require the same final state and
statistics every time. usage: python scripts/repeat_check.py <config> <reps> [key=value ...]
(values are Python literals, e.g. shards=4 early_reject=1 dims=(2048,2048) T=5.0)"""
import ast
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_cs_0502039_b200 as aca  # noqa: E402
import workloads  # noqa: E402

name, reps = sys.argv[1], int(sys.argv[2])
cfg = workloads.config(name)
opts = dict(cfg.get("opts", {}))
for kv in sys.argv[3:]:
    k, v = kv.split("=", 1)
    v = ast.literal_eval(v)
    if k in ("dims", "T", "beta", "h", "rule", "init_q"):
        cfg[k] = v
    else:
        opts[k] = v
g = aca.Sim(tuple(cfg["dims"]), lam=cfg["lam"], beta=cfg["beta"], J=cfg["J"], h=cfg["h"], rule=cfg["rule"], seed=2,
            init_q=cfg["init_q"], **opts)
ref, bad = None, 0
for r in range(reps):
    g.reset(2)
    g.run_until(cfg["T"])
    st = g.stats()
    h = hashlib.sha256(g.times().tobytes() + g.spins().tobytes()).hexdigest()[:16]
    got = (st["arrivals"], st["cells_fired"], st["event_hash"], st["bond_sum"], h)
    ok = got[0] == got[1] and (ref is None or got == ref)
    if ref is None:
        ref = got
    if not ok:
        bad += 1
        print("MISMATCH rep", r, got, ref, flush=True)
print(name, opts, "reps", reps, "bad", bad, ref[:2])
