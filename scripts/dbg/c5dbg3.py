import sys, time
sys.path.insert(0, '.')
import torch
import paper_cs_0502039_b200 as aca
dims = (8192, 8192)
use_stream = int(sys.argv[1])
kw = {}
if use_stream:
    stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); kw["stream"] = stream.cuda_stream
g = aca.Sim(dims, beta=1.0, h=0.1, rule=1, init_q=0.05, seed=1, early_reject=1, **kw)
for seed in [1001, 1002, 1003, 1, 2, 3, 4, 5]:
    try:
        g.reset(seed)
        g.run_until(200.0)
        print(seed, "ok", g.stats()["arrivals"], flush=True)
    except Exception as e:
        print(seed, "FAIL", e, flush=True)
        break
