import sys, time
sys.path.insert(0, '.')
import paper_cs_0502039_b200 as aca
dims = tuple(int(x) for x in sys.argv[1].split('x'))
early = int(sys.argv[2])
g = aca.Sim(dims, beta=1.0, h=0.1, rule=1, init_q=0.05, seed=1, early_reject=early)
for T in [float(x) for x in sys.argv[3].split(',')]:
    t0 = time.time()
    try:
        g.run_until(T)
        st = g.stats()
        print(dims, early, T, "ok", st["arrivals"], st["counter_bits"], "%.2fs" % (time.time() - t0), flush=True)
    except Exception as e:
        print(dims, early, T, "FAIL", e, flush=True)
        break
