import os, sys, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_cs_0502039_b200 as aca, workloads
name = sys.argv[1]; seed = int(sys.argv[2])
cfg = workloads.config(name)
g = aca.Sim(cfg["dims"], lam=cfg["lam"], beta=cfg["beta"], J=cfg["J"], h=cfg["h"], rule=cfg["rule"], seed=seed,
            init_q=cfg["init_q"], **cfg.get("opts", {}))
g.run_until(cfg["T"])
st = g.stats()
tot = int(g.counters().astype(np.int64).sum())
print(name, seed, os.environ.get("ACA_NO_TMA_BOX"), tot, st["arrivals"], st["cells_fired"], tot - st["cells_fired"], st["launches"])
