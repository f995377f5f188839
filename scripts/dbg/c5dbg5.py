import sys, json
sys.path.insert(0, '.')
import torch
import paper_cs_0502039_b200 as aca
dims = tuple(int(x) for x in sys.argv[1].split('x'))
kw = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
phys = dict(beta=1.0, h=0.1, rule=1, init_q=0.05)
phys.update(kw.pop("phys", {}))
T = kw.pop("T", 200.0)
g = aca.Sim(dims, seed=kw.pop("seed", 1001), early_reject=kw.pop("early_reject", 1), **phys, **kw)
try:
    g.run_until(T)
    print(sys.argv[1:], "ok", g.stats()["arrivals"], flush=True)
except Exception as e:
    print(sys.argv[1:], "FAIL", e, flush=True)
