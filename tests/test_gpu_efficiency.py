"""GPU time-only efficiency model through the C ABI: bit-identical to the
oracle's iterations (every N0 and every final time) on small arrays, and at sizes far beyond
the oracle's reach the steady-state efficiency equals the values the paper prints
(tests/golden/paper_efficiency.txt)."""
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dims", [(2,), (37,), (1000,), (2, 2), (13, 7), (64, 48), (2, 2, 2), (12, 10, 8)])
@pytest.mark.parametrize("law", [0, 1, 2, 3])
def test_efficiency_bit_identical(aca, oracle_mod, dims, law):
    rounds = 150
    f_g, t_g, _ = aca.aca_efficiency_run(dims, rounds, law=law, seed=31, want_times=True)
    f_o, t_o = oracle_mod.efficiency_run(dims, rounds, law=law, seed=31, want_times=True)
    assert np.array_equal(f_g, f_o)
    assert np.array_equal(t_g, t_o)


def _golden():
    rows = []
    for line in open(os.path.join(HERE, "golden", "paper_efficiency.txt")):
        if not line.startswith("#") and line.strip():
            nd, law, v, tol = line.split()
            rows.append((int(nd), int(law), float(v), float(tol)))
    return rows


@pytest.mark.parametrize("ndim,law,value,tol", _golden())
def test_efficiency_large_arrays_match_paper(aca, ndim, law, value, tol):
    """1-D n = 2^24, 2-D 4096 x 4096: 400 iterations, the last 250 averaged."""
    dims = (1 << 24,) if ndim == 1 else (4096, 4096)
    fired, _ = aca.aca_efficiency_run(dims, 400, law=law, seed=101 + law)
    eff = fired[150:].astype(np.float64) / np.prod(dims)
    assert abs(eff.mean() - value) < tol, (eff.mean(), value)


def test_efficiency_rejects_bad_arguments(aca):
    for dims, law in (((1,), 0), ((4, 4), 4)):
        with pytest.raises(aca.AcaError):
            aca.aca_efficiency_run(dims, 5, law=law)


@pytest.mark.parametrize("dims", [(9,), (1000,), (40, 30), (13, 7), (10, 8, 6)])
@pytest.mark.parametrize("q", [2, 3])
def test_efficiency_q_bit_identical(aca, oracle_mod, dims, q):
    """q-th degree neighbourhood (Eq. neiq): every N0 and final time."""
    f_g, t_g, _ = aca.aca_efficiency_run(dims, 80, law=0, seed=41, want_times=True, q=q)
    f_o, t_o = oracle_mod.efficiency_run(dims, 80, law=0, seed=41, want_times=True, q=q)
    assert np.array_equal(f_g, f_o) and np.array_equal(t_g, t_o)


@pytest.mark.parametrize("dims", [(700, 300), (256, 64), (257, 65), (33, 130)])
def test_efficiency_2d_streaming_kernel(aca, oracle_mod, dims):
    """The 2-D row-streaming kernel (strips of 256 columns, bands of 64 rows, partial strips and
    bands, halo columns across strips and the periodic wrap) equals the oracle."""
    f_g, t_g, _ = aca.aca_efficiency_run(dims, 60, law=1, seed=43, want_times=True)
    f_o, t_o = oracle_mod.efficiency_run(dims, 60, law=1, seed=43, want_times=True)
    assert np.array_equal(f_g, f_o) and np.array_equal(t_g, t_o)


@pytest.mark.parametrize("px,py,m,lag,rounds", [(5, 5, 24, 0.0, 3000), (32, 32, 12, 0.3, 1500), (32, 32, 12, 16.0, 1500),
                                               (7, 3, 2, 0.0, 500), (100, 100, 100, 0.0, 300), (1, 1, 12, 0.0, 50),
                                               (6, 5, 12, 1.0 / 2 ** 32, 400)])
def test_perfbl_model_bit_identical_to_oracle(aca, oracle_mod, px, py, m, lag, rounds):
    """fig:perfbl model (P11): the GPU's per-round advance counts and final (h, n) equal the
    oracle's, including the paper's configurations (25 PEs / m = 24; 1024 PEs / m = 12 with a lag
    bound; 10^4 PEs / m = 100)."""
    ug, hg, ng = aca.aca_perfbl_run(px, py, m, rounds, lag=lag, seed=4)
    uo, ho, no = oracle_mod.perfbl_run(px, py, m, rounds, lag=lag, seed=4)
    assert np.array_equal(ug, uo) and np.array_equal(hg, ho) and np.array_equal(ng, no)
