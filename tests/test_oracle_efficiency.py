"""Pins of the oracle's time-only efficiency model against the values
the paper prints (tests/golden/paper_efficiency.txt) and against exact special cases."""
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def _golden():
    rows = []
    for line in open(os.path.join(HERE, "golden", "paper_efficiency.txt")):
        if line.startswith("#") or not line.strip():
            continue
        nd, law, v, tol = line.split()
        rows.append((int(nd), int(law), float(v), float(tol)))
    return rows


@pytest.mark.parametrize("ndim,law,value,tol", _golden())
def test_efficiency_matches_paper(oracle_mod, ndim, law, value, tol):
    """Steady-state N0/N of a large array (1-D n = 40000, 2-D 200 x 200), averaged over
    iterations after a warm-up, equals the paper's limiting value within its precision."""
    dims = (40000,) if ndim == 1 else (200, 200)
    fired = oracle_mod.efficiency_run(dims, 700, law=law, seed=11 + law)
    eff = fired[200:].astype(np.float64) / np.prod(dims)
    assert abs(eff.mean() - value) < tol, (eff.mean(), value)


def test_efficiency_two_cell_circle(oracle_mod):
    """n = 2: the two cells are each other's neighbours (twice); exactly the smaller (t, c)
    fires each iteration, so N0 = 1 always (efficiency exactly 1/2)."""
    for law in (0, 1, 2):
        fired = oracle_mod.efficiency_run((2,), 200, law=law, seed=3)
        assert np.all(fired == 1)


def test_efficiency_invariants(oracle_mod):
    """Every iteration fires >= 1 cell (the global minimum) and at most an independent set
    (<= N/2 on a bipartite torus); times only grow, and cells that fired k times sit at the
    sum of k increments (checked through the total: sum of N0 = number of increments)."""
    for dims in ((64,), (16, 12), (6, 4, 8)):
        n = int(np.prod(dims))
        fired, t = oracle_mod.efficiency_run(dims, 300, law=0, seed=5, want_times=True)
        assert fired.min() >= 1 and fired.max() <= n // 2
        fired0, t0 = oracle_mod.efficiency_run(dims, 0, law=0, seed=5, want_times=True)
        assert np.all(t >= t0) and int((t > t0).sum()) <= n


def test_efficiency_rate_invariance(oracle_mod):
    """Scaling every increment by 1/lambda does not change which cells pass the test, so the
    N0 sequence is the same for every lambda whose scaling keeps the order (lambda = 1/2
    doubles every increment exactly)."""
    a = oracle_mod.efficiency_run((32, 32), 100, law=1, lam=1.0, seed=9)
    b = oracle_mod.efficiency_run((32, 32), 100, law=1, lam=0.5, seed=9)
    assert np.array_equal(a, b)


def _neighbors_q(q, L=31):
    """Eq. neiq taken literally on an L x L torus: neighbors^1(c) = c and
    its 4 neighbours; neighbors^q = neighbors(neighbors^(q-1))."""
    def nb(c):
        x, y = c
        return {c, ((x - 1) % L, y), ((x + 1) % L, y), (x, (y - 1) % L), (x, (y + 1) % L)}
    S = {(0, 0)}
    for _ in range(q):
        S = set().union(*(nb(c) for c in S))
    return S


@pytest.mark.parametrize("q", [1, 2, 3, 4])
def test_neighbourhood_q_definition(q):
    """|neighbors^q(c)| - 1 = 2q(q+1), and the set is exactly the cells
    within Manhattan distance q — the set the oracle's test loops over."""
    S = _neighbors_q(q)
    assert len(S) - 1 == 2 * q * (q + 1)
    L = 31
    diamond = {((dx) % L, (dy) % L) for dx in range(-q, q + 1) for dy in range(-q, q + 1) if abs(dx) + abs(dy) <= q}
    assert S == diamond


def test_efficiency_q_special_cases(oracle_mod):
    """q = 1 is the plain model; an n-circle with q >= (n-1)/2 is one neighbourhood, so exactly
    the global minimum fires each iteration; efficiency falls with q ("low efficiency",
    PAPER.md:1011-1020)."""
    a = oracle_mod.efficiency_run((40, 30), 120, seed=4)
    b = oracle_mod.efficiency_run((40, 30), 120, seed=4, q=1)
    assert np.array_equal(a, b)
    for n, q in ((9, 4), (10, 5), (5, 2)):
        assert set(oracle_mod.efficiency_run((n,), 80, seed=2, q=q).tolist()) == {1}
    effs = [oracle_mod.efficiency_run((96, 96), 300, seed=6, q=q)[100:].mean() / 96 ** 2 for q in (1, 2, 3)]
    assert effs[0] > effs[1] > effs[2] > 0
