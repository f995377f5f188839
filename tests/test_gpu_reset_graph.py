"""aca_reset keeps the instantiated CUDA graph of the tile launches and updates its parameters
(the new seed's Philox round keys) in place at the next run_until (cudaGraphExecUpdate) instead of
re-instantiating it. Every run after a reset must equal the serial oracle for that seed, whatever
the previous seed, horizon or kernel instance was."""
import numpy as np
import pytest

from test_gpu_parity import aca, assert_same  # noqa: F401  (fixture + helpers)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dims,phys,opts", [
    ((200, 136), dict(beta=0.4406868, rule=0), dict(whole_lattice=-1)),
    ((40, 36, 20), dict(beta=0.2216544, rule=0), dict(whole_lattice=-1)),
    ((256, 192), dict(beta=1.0, h=0.1, rule=1, init_q=0.05), dict(early_reject=1, class_book=1, class_wmax=0.01)),
])
def test_reset_reuses_graph(aca, oracle_mod, dims, phys, opts):
    g = aca.Sim(dims, seed=1, **phys, **opts)
    seq = [(1, 4.0), (7, 4.0), (7, 6.0), (3, 3.0), (1, 5.0)]   # (seed, T); same seed twice = a plain reset
    for seed, T in seq:
        g.reset(seed)
        g.run_until(T)
        o = oracle_mod.OracleSim(dims, seed=seed, **phys)
        o.run_until(T)
        assert_same(g, o)
    g.close()
