"""The resident-tile kernel (res_kernel, csrc/aca_res.cuh): small 2-D lattices whose 64 x 64 tiles
fit in the SMs' shared memory run a whole run_until in one cooperative launch, tiles resident
across sweeps, grid barriers between the checkerboard colours. Same schedule family as the tile
kernel, so the trajectory must be the oracle's, bit for bit."""
import numpy as np
import pytest

from test_gpu_parity import aca, assert_same, run_pair  # noqa: F401  (fixture + helpers)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dims,Ts,kw", [
    ((128, 128), [5.0], dict(beta=0.4406868)),                        # 4 tiles: 2 CTAs
    ((256, 192), [3.0, 7.5], dict(beta=0.4406868)),                   # odd tile rows, composition
    ((192, 320), [6.0], dict(beta=0.40, rule=1)),                     # odd tile counts (wrap neighbours)
    ((1024, 512), [4.0], dict(beta=1.0, h=0.1, rule=1, init_q=0.05)),  # 128 tiles
    ((1024, 1024), [3.0], dict(beta=0.40, rule=1)),                   # config 2's lattice: 128 CTAs
    ((1536, 1536), [2.0], dict(beta=0.4406868)),                      # 288 tiles: two per colour per CTA
])
def test_resident_kernel_exact(aca, oracle_mod, dims, Ts, kw):
    g, o = run_pair(aca, oracle_mod, dims, Ts, seed=71, whole_lattice=-1, **kw)
    assert_same(g, o)
    assert g.stats()["kernel_launches"] <= 2 * len(Ts), "the resident path: one launch (+ a no-op) per run_until"


def test_resident_equals_tile_kernel(aca, monkeypatch):
    """The same run through the resident kernel and the grouped tile kernel (ACA_NO_RES=1)."""
    dims = (512, 512)
    a = aca.Sim(dims, beta=0.4406868, seed=5, whole_lattice=-1)
    a.run_until(6.0)
    monkeypatch.setenv("ACA_NO_RES", "1")
    b = aca.Sim(dims, beta=0.4406868, seed=5, whole_lattice=-1)
    b.run_until(6.0)
    assert a.stats()["kernel_launches"] < b.stats()["kernel_launches"]
    for f in ("spins", "times", "counters"):
        assert np.array_equal(getattr(a, f)(), getattr(b, f)())
    sa, sb = a.stats(), b.stats()
    for k in ("arrivals", "flips", "event_hash", "bond_sum", "magnetisation"):
        assert sa[k] == sb[k]


def test_resident_falls_back(aca, oracle_mod):
    """Runs the resident kernel does not take (ties, lag window) still match."""
    g, o = run_pair(aca, oracle_mod, (256, 256), [4.0], seed=9, whole_lattice=-1, tie_bits=30)
    assert_same(g, o)
    g, o = run_pair(aca, oracle_mod, (256, 256), [4.0], seed=9, whole_lattice=-1, lag=0.5)
    assert_same(g, o)
