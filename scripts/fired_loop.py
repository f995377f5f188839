"""Repeat a config's run and compare sum n(c) with the kernels' fired count and a reference total
(race hunting). usage: python scripts/fired_loop.py c3 <seed> <reps>"""
import os, sys, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_cs_0502039_b200 as aca, workloads
name, seed, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
cfg = workloads.config(name)
g = aca.Sim(cfg["dims"], lam=cfg["lam"], beta=cfg["beta"], J=cfg["J"], h=cfg["h"], rule=cfg["rule"], seed=seed,
            init_q=cfg["init_q"], tile=cfg["tile"], **cfg.get("opts", {}))
ref = None
bad = 0
for r in range(reps):
    g.reset(seed)
    g.run_until(cfg["T"])
    st = g.stats()
    h = st["event_hash"]
    tot = st["arrivals"]
    if ref is None:
        ref = (tot, h, st["cells_fired"])
    ok = (tot, h, st["cells_fired"]) == ref and tot == st["cells_fired"]
    bad += not ok
    if not ok:
        print("MISMATCH rep", r, tot, st["cells_fired"], h, ref, flush=True)
print(name, seed, "box" if not os.environ.get("ACA_NO_TMA_BOX") else "rows", "reps", reps, "bad", bad, ref)
