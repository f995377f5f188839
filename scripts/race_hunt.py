"""Repeat a run until the final state differs from the first run's, then describe the differing
cells (race hunting). usage: python scripts/race_hunt.py c3 <seed> <reps>"""
import os, sys, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_cs_0502039_b200 as aca, workloads
name, seed, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
cfg = workloads.config(name)
g = aca.Sim(cfg["dims"], lam=cfg["lam"], beta=cfg["beta"], J=cfg["J"], h=cfg["h"], rule=cfg["rule"], seed=seed,
            init_q=cfg["init_q"], tile=cfg["tile"], **cfg.get("opts", {}))
ref = None
T = cfg["T"]
for r in range(reps):
    g.reset(seed)
    g.run_until(T)
    st = g.stats()
    if ref is None:
        ref = (g.times().copy(), g.counters().copy(), g.spins().copy(), st["arrivals"])
        continue
    if st["arrivals"] == ref[3]:
        continue
    t, n, s = g.times(), g.counters(), g.spins()
    bad = np.argwhere((t != ref[0]) | (n != ref[1]) | (s != ref[2]))
    print("rep", r, "arrivals", st["arrivals"], "ref", ref[3], "cells differing", len(bad))
    for c in bad[:40]:
        c = tuple(c)
        y, x = c[0], c[1]
        print(" cell y=%d x=%d  tile (%d,%d) local (%d,%d)  t %d -> %d  n %d -> %d  s %d -> %d" % (
            y, x, y // 64, x // 64, y % 64, x % 64, ref[0][c], t[c], ref[1][c], n[c], ref[2][c], s[c]))
    # is the bad value some other cell's reference value?
    for c in bad[:10]:
        c = tuple(c)
        m = np.argwhere((ref[0] == t[c]) & (ref[1] == n[c]))
        print(" value of", c, "matches reference cells", [tuple(v) for v in m[:3]])
    break
print("done")
