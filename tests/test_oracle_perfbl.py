"""The fig:perfbl model in the oracle (docs/PRIMITIVES.md P11)
pinned to what the paper prints (tests/golden/paper_perfbl.txt) and to closed forms:
  * a single PE (its neighbours are itself) advances every round;
  * with a lag window of one Q32 unit only the PEs at the global minimum advance, so the model
    is the serial event-list simulation of the PE streams: its state after R rounds equals a
    brute-force priority queue's after R pops (independent of the neighbour checks, which the
    minimum always passes);
  * very large subarrays (p0 -> 1) run at efficiency -> 1."""
import heapq
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "paper_perfbl.txt")


def paper():
    d = {}
    for ln in open(GOLD):
        if ln.strip() and not ln.startswith("#"):
            k, v = ln.split()[:2]
            d[k] = float(v)
    return d


def eff(oracle_mod, px, py, m, rounds, lag=0.0, seeds=(1,), warm=0.25):
    out = []
    for s in seeds:
        ups, _, _ = oracle_mod.perfbl_run(px, py, m, rounds, lag=lag, seed=s)
        out.append(ups[int(rounds * warm):].mean() / (px * py))
    return float(np.mean(out))


def test_paper_efficiencies_of_the_model(oracle_mod):
    p = paper()
    e25 = eff(oracle_mod, 5, 5, 24, 20000, seeds=(1, 2, 3, 4))
    assert abs(e25 - p["eff_25pe_m24_n120"]) < 0.03, e25
    e4 = eff(oracle_mod, 100, 100, 100, 1200)
    assert abs(e4 - p["eff_1e4pe_m100"]) < 0.02, e4


def test_paper_lag_degradation_shape(oracle_mod):
    """fig:perfbl: n = 384, m = 12, i.e. 32 x 32 = 1024 PEs; lag in units of a cell's mean
    inter-arrival time."""
    p = paper()
    base = eff(oracle_mod, 32, 32, 12, 4000)
    e16 = eff(oracle_mod, 32, 32, 12, 4000, lag=16.0)
    e8 = eff(oracle_mod, 32, 32, 12, 4000, lag=8.0)
    e4 = eff(oracle_mod, 32, 32, 12, 4000, lag=4.0)
    e1 = eff(oracle_mod, 32, 32, 12, 4000, lag=1.0)
    e03 = eff(oracle_mod, 32, 32, 12, 4000, lag=0.3)
    assert abs(e16 / base - p["lag16_rel"]) < 0.02                 # almost unnoticeable
    assert e4 < 0.95 * base and e8 <= e16 + 0.005                  # degradation sets in below ~8
    assert abs(e1 / base - p["lag1_rel"]) < 0.1                    # about half
    assert abs(e03 - p["lag03_eff"]) < 0.05 and e03 * 1024 > 100   # about 0.1, speed-up > 100
    assert base > e16 - 0.005 > e4 > e1 > e03


def test_single_pe_always_advances(oracle_mod):
    ups, h, n = oracle_mod.perfbl_run(1, 1, 12, 500, seed=5)
    assert (ups == 1).all() and int(n[0]) == 500


def test_unit_lag_is_the_serial_event_order(oracle_mod):
    """lag = 1 Q32 unit: a round advances exactly the PEs at the snapshot minimum; the state after
    R rounds is the serial simulation of the PE streams (priority queue on (h, C))."""
    px, py, m, R, seed = 6, 5, 12, 400, 9
    ups, h, n = oracle_mod.perfbl_run(px, py, m, R, lag=1.0 / 2 ** 32, seed=seed)
    key = (seed & 0xFFFFFFFF, seed >> 32)

    def inc(ctr):
        w = oracle_mod.philox(ctr, key)
        return max(1, oracle_mod.nlog_q32((w[2] << 32) | w[3]))

    N = px * py
    hh = [inc((0, C, 0, 8)) for C in range(N)]
    nn = [0] * N
    pq = [(hh[C], C) for C in range(N)]
    heapq.heapify(pq)
    for r in range(R):   # one pop per round unless several PEs share the minimum (then all of them)
        t0 = pq[0][0]
        popped = []
        while pq and pq[0][0] == t0:
            popped.append(heapq.heappop(pq))
        assert int(ups[r]) == len(popped)
        for t, C in popped:
            hh[C] = t + inc((nn[C], C, 0, 7))
            nn[C] += 1
            heapq.heappush(pq, (hh[C], C))
    assert list(h) == hh and list(n) == nn


def test_large_subarrays_run_at_full_efficiency(oracle_mod):
    """p0 = (m-2)^2/m^2 -> 1: the efficiency rises with m towards 1."""
    e = [eff(oracle_mod, 8, 8, m, 2000) for m in (12, 100, 1000, 65535)]
    assert e[0] < e[1] < e[2] < e[3] and e[3] > 0.995, e


def test_invariants(oracle_mod):
    for px, py, m, lag in ((7, 3, 2, 0.0), (4, 9, 5, 2.0), (16, 16, 24, 0.5)):
        ups, h, n = oracle_mod.perfbl_run(px, py, m, 300, lag=lag, seed=3)
        assert (ups <= px * py).all() and int(n.sum()) == int(ups.sum())
        _, h0, _ = oracle_mod.perfbl_run(px, py, m, 0, seed=3)
        assert (h >= h0).all()
