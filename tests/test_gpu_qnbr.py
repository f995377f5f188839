"""The Ising model on the q-th degree neighbourhood (Eq. neiq; docs/PRIMITIVES.md
P12) on the GPU through the C ABI: bit-identical to the serial oracle (spins, every t(c), every
n(c), arrivals, flips, event hash, B, M) for q = 1..4 in 2-D and 3-D, ragged tiles, odd tile counts
(three colours per axis), the smallest sides (2q + 1), forced ties, both rules, a field, lambda != 1,
other asynchrony laws and one round per visit; q = 1 is the main path's trajectory."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _pair(aca, oracle_mod, dims, q, T, **kw):
    rounds = kw.pop("rounds", 0)
    g = aca.aca_qnbr_run(dims, q, T, rounds=rounds, **kw)
    o = oracle_mod.OracleSim(dims, q=q, **kw)
    o.run_until(T)
    return g, o


def _same(g, o):
    gs, gt, gn, gst = g
    assert np.array_equal(gs, o.spins()), "spins"
    assert np.array_equal(gt, o.times()), "times"
    assert np.array_equal(gn, o.counters()), "counters"
    ost = o.stats()
    for k in ("arrivals", "flips", "event_hash", "bond_sum", "magnetisation"):
        assert gst[k] == ost[k], (k, gst[k], ost[k])
    assert gst["arrivals"] > 0


@pytest.mark.parametrize("dims,q", [((16, 16), 2), ((37, 29), 3), ((69, 70), 2), ((128, 96), 4), ((5, 5), 2),
                                    ((9, 11), 4), ((200, 136), 2), ((96, 97), 3), ((64, 64), 1)])
@pytest.mark.parametrize("rule", [0, 1])
def test_qnbr_2d_bit_identical(aca, oracle_mod, dims, q, rule):
    kw = dict(beta=0.12 if rule == 0 else 0.3, h=0.0 if rule == 0 else 0.1, rule=rule, seed=11 + q)
    _same(*_pair(aca, oracle_mod, dims, q, 6.0, **kw))


@pytest.mark.parametrize("dims,q", [((9, 10, 11), 2), ((20, 18, 17), 3), ((5, 5, 6), 2), ((24, 16, 9), 4),
                                    ((33, 17, 16), 2), ((16, 16, 16), 1)])
def test_qnbr_3d_bit_identical(aca, oracle_mod, dims, q):
    _same(*_pair(aca, oracle_mod, dims, q, 4.0, beta=0.08, seed=21 + q))


@pytest.mark.parametrize("dims,q,tie_bits", [((64, 48), 2, 28), ((33, 35), 3, 27), ((12, 11, 10), 2, 28),
                                             ((40, 40), 4, 29)])
def test_qnbr_forced_ties(aca, oracle_mod, dims, q, tie_bits):
    _same(*_pair(aca, oracle_mod, dims, q, 5.0, beta=0.2, tie_bits=tie_bits, seed=5))


@pytest.mark.parametrize("law", [1, 2, 3])
def test_qnbr_laws(aca, oracle_mod, law):
    _same(*_pair(aca, oracle_mod, (70, 66), 2, 5.0, beta=0.15, law=law, seed=8))


def test_qnbr_lambda_field_init_rounds(aca, oracle_mod):
    _same(*_pair(aca, oracle_mod, (100, 90), 2, 3.0, lam=2.5, beta=0.5, h=-0.3, rule=1, init_q=0.05, seed=4))
    _same(*_pair(aca, oracle_mod, (100, 90), 3, 4.0, beta=0.1, seed=4, rounds=1))


def test_qnbr_q1_is_the_main_path(aca, oracle_mod):
    dims = (96, 80)
    g = aca.aca_qnbr_run(dims, 1, 5.0, beta=0.4406868, seed=3)
    s = aca.Sim(dims, beta=0.4406868, seed=3, device=0)
    s.run_until(5.0)
    assert np.array_equal(g[0], s.spins()) and np.array_equal(g[1], s.times()) and np.array_equal(g[2], s.counters())
    assert g[3]["event_hash"] == s.stats()["event_hash"]
    s.close()


def test_qnbr_large_lattice(aca, oracle_mod):
    """2048^2 with q = 2 (4096 tiles, 4 colours) against the full oracle."""
    _same(*_pair(aca, oracle_mod, (2048, 2048), 2, 3.0, beta=0.1, seed=7))


def test_qnbr_argument_errors(aca):
    for dims, q in (((4, 9), 2), ((9, 9), 5), ((9, 9), 0), ((9,), 1)):
        with pytest.raises(aca.AcaError):
            aca.aca_qnbr_run(dims, q, 1.0)
