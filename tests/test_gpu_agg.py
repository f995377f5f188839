"""Aggregated Poisson stream (fig:amcpoi) on the GPU through the C ABI:
bit-identical to the serial oracle for the same partition (spins, every T(C), every n(C),
arrivals, flips, event hash, B, M), across subarray sizes, rules, launch budgets (small
budgets force many blocked/resumed launches) and lattices one or two subarrays wide; m = 1
reproduces the main path's trajectory."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _same(g, o):
    gs, gT, gn, gst = g
    os_, oT, on, ost = o
    assert np.array_equal(gs, os_)
    assert np.array_equal(gT, oT) and np.array_equal(gn, on)
    for k in ("arrivals", "flips", "event_hash", "bond_sum", "magnetisation"):
        assert gst[k] == ost[k], (k, gst[k], ost[k])


@pytest.mark.parametrize("dims,m", [((64, 64), 8), ((64, 48), 4), ((40, 24), 2), ((16, 16), 1), ((8, 8), 8),
                                    ((16, 8), 8), ((12, 6), 2), ((256, 128), 8), ((9, 6), 3), ((48, 36), 12),
                                    ((120, 120), 24), ((384, 384), 12), ((96, 64), 32)])
@pytest.mark.parametrize("rule", [0, 1])
def test_agg_bit_identical(aca, oracle_mod, dims, m, rule):
    kw = dict(beta=0.44 if rule == 0 else 0.6, h=0.0 if rule == 0 else 0.1, rule=rule, seed=5 + m)
    g = aca.aca_agg_run(dims, m, 6.0, budget=16, **kw)
    o = oracle_mod.agg_run(dims, m, 6.0, **kw)
    _same(g, o)


@pytest.mark.parametrize("budget", [1, 3, 1000])
def test_agg_budget_invariance(aca, oracle_mod, budget):
    g = aca.aca_agg_run((96, 64), 4, 5.0, beta=0.44, seed=77, budget=budget)
    o = oracle_mod.agg_run((96, 64), 4, 5.0, beta=0.44, seed=77)
    _same(g, o)


def test_agg_m1_equals_main_path(aca, oracle_mod):
    g = aca.aca_agg_run((48, 32), 1, 4.0, beta=0.44, seed=3)
    s = aca.Sim((48, 32), beta=0.44, seed=3, whole_lattice=-1)
    s.run_until(4.0)
    assert np.array_equal(g[0], s.spins())
    assert np.array_equal(g[1], s.times().ravel()) and np.array_equal(g[2], s.counters().ravel())
    assert g[3]["event_hash"] == s.stats()["event_hash"]


def test_agg_rejects_bad_arguments(aca):
    for dims, m in (((10, 8), 4), ((8, 8), 3), ((8, 8), 16), ((66, 66), 33)):
        with pytest.raises(aca.AcaError):
            aca.aca_agg_run(dims, m, 1.0)


@pytest.mark.parametrize("dims,m", [((64, 64), 8), ((64, 48), 4), ((40, 24), 2), ((8, 8), 8), ((16, 8), 8),
                                    ((256, 128), 8), ((4, 4), 4), ((9, 6), 3), ((48, 36), 12), ((120, 120), 24),
                                    ((96, 64), 32)])
@pytest.mark.parametrize("rule", [0, 1])
def test_bkl_bit_identical(aca, oracle_mod, dims, m, rule):
    """Modified BKL: bit-identical to its serial oracle for the partition."""
    kw = dict(beta=0.44 if rule == 0 else 0.9, h=0.0 if rule == 0 else 0.1, rule=rule, seed=11 + m)
    g = aca.aca_agg_run(dims, m, 6.0, budget=16, bkl=True, **kw)
    o = oracle_mod.agg_run(dims, m, 6.0, bkl=True, **kw)
    _same(g, o)


@pytest.mark.parametrize("budget", [1, 1000])
def test_bkl_budget_invariance(aca, oracle_mod, budget):
    g = aca.aca_agg_run((96, 64), 8, 5.0, beta=0.6, rule=1, h=0.1, seed=78, budget=budget, bkl=True)
    o = oracle_mod.agg_run((96, 64), 8, 5.0, beta=0.6, rule=1, h=0.1, seed=78, bkl=True)
    _same(g, o)
