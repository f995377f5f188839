"""Asynchronous Game of Life (rule 2, P10): Conway's B3/S23 rule applied at
each cell's Poisson arrivals, Moore neighbourhood. Pins: still lifes and a lone cell behave as
the rule dictates under any order; the trajectory is unique (PQ = random order = synchronous
rounds, with and without forced time ties); it does not depend on beta, J, h (deterministic)."""
import numpy as np
import pytest

LIFE = 2


def test_life_block_is_still(oracle_mod):
    """A 2x2 block on an empty torus: every live cell has 3 live neighbours (stays), every dead
    cell at most 2 (stays dead) — no arrival changes anything."""
    o = oracle_mod.OracleSim((12, 10), rule=LIFE, seed=3)
    s = -np.ones((10, 12), np.int8)
    s[4:6, 5:7] = 1
    o.set_spins(s)
    o.run_until(20.0)
    assert np.array_equal(o.spins(), s) and o.stats()["flips"] == 0 and o.stats()["arrivals"] > 2000


def test_life_lone_cell_dies_alone(oracle_mod):
    """One live cell: it dies at its first arrival (0 live neighbours), no dead cell ever sees 3
    live neighbours, so exactly one flip happens."""
    o = oracle_mod.OracleSim((9, 7), rule=LIFE, seed=5)
    s = -np.ones((7, 9), np.int8)
    s[3, 4] = 1
    o.set_spins(s)
    o.run_until(10.0)
    assert np.all(o.spins() == -1) and o.stats()["flips"] == 1


@pytest.mark.parametrize("dims", [(16, 16), (5, 7), (2, 6), (3, 3)])
@pytest.mark.parametrize("tie_bits", [0, 30])
def test_life_order_independence(oracle_mod, dims, tie_bits):
    res = []
    for order, cs in (("pq", 0), ("random", 1), ("random", 2), ("sync", 0)):
        o = oracle_mod.OracleSim(dims, rule=LIFE, seed=21, tie_bits=tie_bits, init_q=0.6)
        o.run_until(6.0, order=order, choice_seed=cs)
        st = o.stats()
        st.pop("rounds")
        res.append((o.spins().copy(), o.times().copy(), o.counters().copy(), st))
    for other in res[1:]:
        for a, b in zip(res[0][:3], other[:3]):
            assert np.array_equal(a, b)
        assert res[0][3] == other[3]


def test_life_is_deterministic_in_beta(oracle_mod):
    a = oracle_mod.OracleSim((20, 14), rule=LIFE, seed=8, beta=0.1)
    b = oracle_mod.OracleSim((20, 14), rule=LIFE, seed=8, beta=2.0, h=0.3, J=-1.0)
    a.run_until(8.0)
    b.run_until(8.0)
    assert np.array_equal(a.spins(), b.spins()) and a.stats()["flips"] == b.stats()["flips"] > 0
