import sys, numpy as np
sys.path.insert(0, '.')
import paper_cs_0502039_b200 as aca
import oracle
dims = tuple(int(x) for x in sys.argv[1].split('x'))
mc = int(sys.argv[2]); T = float(sys.argv[3])
g = aca.Sim(dims, beta=1.0, h=0.1, rule=1, init_q=0.05, seed=1, early_reject=1, max_ctas=mc)
g.run_until(T)
print("gpu ok", g.stats()["arrivals"])
if len(sys.argv) > 4:
    o = oracle.OracleSim(dims, beta=1.0, h=0.1, rule=1, init_q=0.05, seed=1)
    o.run_until(T)
    print("spins", np.array_equal(g.spins(), o.spins()), "times", np.array_equal(g.times(), o.times()))
