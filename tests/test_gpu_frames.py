"""Output frames (fig:genout) through the C ABI: the frame for time K dt
equals the oracle's spins after every arrival at or before K dt (run_until(K dt + 1 unit)),
bit for bit, for every window size B (the bounded lag), tile shape / kernel variant, shard
count and law; the run continues exactly afterwards."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def oracle_frames(oracle_mod, dims, dt, K0, count, T_before=None, **kw):
    o = oracle_mod.OracleSim(dims, **kw)
    if T_before is not None:
        o.run_until(T_before)
    dq = int(np.floor(dt * 4294967296.0 + 0.5))
    out = []
    for K in range(K0, K0 + count):
        o.run_until_q32(K * dq + 1)
        out.append(o.spins().copy())
    return np.stack(out), o


@pytest.mark.parametrize("B", [1, 3, 16])
def test_frames_match_oracle(aca, oracle_mod, B):
    dims = (200, 150)
    kw = dict(beta=0.44, seed=29, rule=0)
    g = aca.Sim(dims, whole_lattice=-1, **kw)
    want, o = oracle_frames(oracle_mod, dims, 0.5, 1, 9, **kw)
    got = g.frames(0.5, 1, 9, B=B)
    assert np.array_equal(got, want)
    # the simulation continues exactly after the frames
    g.run_until(7.0)
    o.run_until(7.0)
    assert np.array_equal(g.spins(), o.spins()) and np.array_equal(g.times(), o.times())
    assert g.stats()["event_hash"] == o.stats()["event_hash"]


@pytest.mark.parametrize("case", ["whole", "v0_3d", "early", "shards", "law2", "ties", "after_run"])
def test_frames_variants(aca, oracle_mod, case):
    dims, kw, opts, dt, K0, cnt, Tb = (130, 70), dict(beta=0.44, seed=3), dict(whole_lattice=-1), 0.37, 2, 7, None
    if case == "whole":
        dims, opts = (24, 20), dict(whole_lattice=1)
    elif case == "v0_3d":
        dims, kw, opts = (32, 24, 16), dict(beta=0.22, seed=4), dict(whole_lattice=-1, tile=(16, 16, 16))
    elif case == "early":
        kw, opts = dict(beta=1.0, h=0.1, rule=1, init_q=0.05, seed=5), dict(whole_lattice=-1, early_reject=1)
    elif case == "shards":
        dims, opts = (128, 96), dict(shards=4)
    elif case == "law2":
        kw = dict(beta=0.44, seed=6, law=2)
    elif case == "ties":
        kw = dict(beta=0.44, seed=7, tie_bits=30)
        dt = 0.5                      # frame times coincide with quantised arrival times
    elif case == "after_run":
        Tb, K0 = 2.3, 7               # frames start after a plain run_until
    g = aca.Sim(dims, **kw, **opts)
    if Tb is not None:
        g.run_until(Tb)
    want, _ = oracle_frames(oracle_mod, dims, dt, K0, cnt, T_before=Tb, **kw)
    got = g.frames(dt, K0, cnt, B=3)
    assert np.array_equal(got.reshape(want.shape), want)


def test_frames_reject_past(aca):
    g = aca.Sim((64, 64), beta=0.44, seed=1, whole_lattice=-1)
    g.run_until(3.0)
    with pytest.raises(aca.AcaError):
        g.frames(1.0, 1, 2)          # frame time 1.0 is already in the past
    with pytest.raises(aca.AcaError):
        g.frames(1.0, 5, 2, B=0)
