import sys, time
sys.path.insert(0, '.')
import torch
import paper_cs_0502039_b200 as aca
dims = tuple(int(x) for x in sys.argv[1].split('x'))
early = int(sys.argv[2])
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
g = aca.Sim(dims, beta=1.0, h=0.1, rule=1, init_q=0.05, seed=1, early_reject=early, stream=stream.cuda_stream)
for seed in [1001, 1002, 1003, 1, 2, 3, 4, 5, 6, 7]:
    try:
        g.reset(seed)
        g.run_until(200.0)
        print(dims, early, seed, "ok", g.stats()["arrivals"], flush=True)
    except Exception as e:
        print(dims, early, seed, "FAIL", e, flush=True)
        break
