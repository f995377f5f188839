"""Equal high halves on the production kernels' fast paths, at small sizes.

The tile kernels decide on the 32-bit high halves of the packed words (t | n | s) and settle equal
high halves in exact passes (strict rounds defer them). On full-size lattices those ties come
from times within 2^(32 - TSH) units of each other (a few dozen per c3/c5 run); on the small
lattices the oracle finishes quickly they almost never occur. ACA_NB_CAP (read by the library
for tests only) narrows the counter field, which widens the high halves' time quantum to
2^-(NB_CAP + 1) time units, so ties are frequent. Every kernel family that runs the fast arrival
must still equal the serial oracle bit for bit (PAPER.md:596-613 uniqueness; lexicographic (t, c)
order, north_star)."""
import pytest

from test_gpu_parity import aca, assert_same, run_pair  # noqa: F401  (fixture + helpers)

pytestmark = pytest.mark.gpu

HB = dict(beta=0.4406868, rule=0)
C5 = dict(beta=1.0, h=0.1, rule=1, init_q=0.05)

CASES = {
    "2d_tile_plain": ((256, 192), [6.0, 12.0], dict(whole_lattice=-1), dict(ACA_NO_RES="1"), HB),
    "2d_resident": ((256, 256), [6.0, 12.0], dict(whole_lattice=-1), {}, HB),
    "2d_capped_ring": ((512, 256), [6.0], dict(max_ctas=3), {}, HB),
    "3d_tile": ((64, 32, 32), [4.0], dict(whole_lattice=-1), {}, dict(beta=0.2216544, rule=0)),
    "3d_a10": ((64, 32, 32), [4.0], dict(whole_lattice=-1, early_reject=1), {}, dict(beta=0.6, h=0.1, rule=1, init_q=0.05)),
    "whole": ((96, 80), [6.0], dict(whole_lattice=1), {}, HB),
    "2d_a10_shards": ((256, 256), [8.0], dict(early_reject=1, shards=2), {}, C5),
    "2d_jacobi": ((256, 192), [6.0], dict(checkerboard=-1, whole_lattice=-1), {}, HB),
}


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("cap", [6, 10])
def test_forced_high_half_ties(aca, oracle_mod, monkeypatch, case, cap):
    dims, Ts, opts, env, phys = CASES[case]
    monkeypatch.setenv("ACA_NB_CAP", str(cap))
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    g, o = run_pair(aca, oracle_mod, dims, Ts, seed=83, **phys, **opts)
    assert_same(g, o)
