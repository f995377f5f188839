"""Pins of the oracle's simulation against what the paper and the mathematics fix:

* state-independence of the arrival times for Ising: every t(c), n(c)
  follows from the cell's own stream alone (a per-cell closed form, no queue);
* beta = 0 closed forms for the spins and m ~ 0 (north_star);
* order independence / uniqueness of the trajectory: PQ order, random
  eligible order and synchronous rounds (fig:s1c1pe) give bit-identical results, also with
  forced ties (P3b);
* run_until composition;
* the stationary distribution = Boltzmann by brute-force enumeration (2x2, 3x3, 2x2x2);
* Onsager's exact 2-D energy per spin (textbook closed form).
"""
import itertools
import math

import mpmath
import numpy as np
import pytest
from scipy import stats as sstats


def closed_form_t_n(oracle_mod, dims, seed, T, lam=1.0, tie_bits=0):
    """Per-cell: t0 = Delta(init draw); while t < T: t += Delta(event draw k), k += 1."""
    N = int(np.prod(dims))
    Tq = oracle_mod.to_q32(T)
    key = (seed & 0xFFFFFFFF, seed >> 32)
    t = np.zeros(N, np.uint64)
    n = np.zeros(N, np.uint32)
    for c in range(N):
        w = oracle_mod.philox((0, c & 0xFFFFFFFF, c >> 32, 1), key)
        tc = oracle_mod.delta(w[1], w[2], lam, tie_bits)
        k = 0
        while tc < Tq:
            w = oracle_mod.philox((k, c & 0xFFFFFFFF, c >> 32, 0), key)
            tc += oracle_mod.delta(w[1], w[2], lam, tie_bits)
            k += 1
        t[c], n[c] = tc, k
    return t.reshape(dims[::-1]), n.reshape(dims[::-1])


@pytest.mark.parametrize("dims,beta,rule,lam,T", [((16, 16), 0.44, 0, 1.0, 7.5), ((5, 7), 1.0, 1, 2.0, 4.0),
                                                  ((2, 2), 0.3, 0, 1.0, 20.0), ((4, 3, 5), 0.22, 0, 0.7, 6.0)])
def test_times_and_counters_closed_form(oracle_mod, dims, beta, rule, lam, T):
    s = oracle_mod.OracleSim(dims, lam=lam, beta=beta, rule=rule, seed=42)
    s.run_until(T)
    t, n = closed_form_t_n(oracle_mod, dims, 42, T, lam)
    assert np.array_equal(s.times(), t)
    assert np.array_equal(s.counters(), n)
    st = s.stats()
    assert st["arrivals"] == int(n.sum())
    assert st["t_min"] >= oracle_mod.to_q32(T)


def test_arrival_count_is_poisson(oracle_mod):
    """Sum n = N lambda T +- 4 sqrt(N lambda T)."""
    for lam, T in ((1.0, 10.0), (3.0, 2.0)):
        s = oracle_mod.OracleSim((64, 64), lam=lam, beta=0.4406868, seed=5)
        s.run_until(T)
        mu = 64 * 64 * lam * T
        assert abs(s.stats()["arrivals"] - mu) < 4 * math.sqrt(mu)


@pytest.mark.parametrize("rule", [0, 1])
def test_beta_zero_spin_closed_form(oracle_mod, rule):
    """beta = 0: Metropolis always flips, s = s0 (-1)^n; heat-bath flips iff w0 < 2^31."""
    dims, seed, T = (9, 11), 77, 6.0
    s = oracle_mod.OracleSim(dims, beta=0.0, rule=rule, seed=seed, h=0.3)
    s.run_until(T)
    n = s.counters().ravel()
    key = (seed, 0)
    exp = np.empty(n.size, np.int8)
    for c in range(n.size):
        w = oracle_mod.philox((0, c, 0, 1), key)
        sc = -1 if w[0] < 2 ** 31 else 1
        for k in range(int(n[c])):
            w = oracle_mod.philox((k, c, 0, 0), key)
            if rule == 1 or w[0] < 2 ** 31:
                sc = -sc
        exp[c] = sc
    assert np.array_equal(s.spins().ravel(), exp)


def test_beta_zero_magnetisation_near_zero(oracle_mod):
    s = oracle_mod.OracleSim((128, 128), beta=0.0, seed=3)
    s.run_until(5.0)
    assert abs(s.stats()["magnetisation"]) < 5 * math.sqrt(128 * 128)


def test_init_rule(oracle_mod):
    """P5: init_q = 0.05 gives i.i.d. Bernoulli(0.05) minority; init_q = 0 gives all +1."""
    s = oracle_mod.OracleSim((256, 256), beta=1.0, rule=1, h=0.1, seed=11, init_q=0.05)
    frac = float((s.spins() < 0).mean())
    assert abs(frac - 0.05) < 5 * math.sqrt(0.05 * 0.95 / 65536)
    s0 = oracle_mod.OracleSim((8, 8), seed=1, init_q=0.0)
    assert (s0.spins() == 1).all()


def _run_all_orders(oracle_mod, dims, T, tie_bits, seed, beta=0.4406868, rule=0, h=0.0, law=0):
    out = []
    for order, cs in (("pq", 0), ("random", 1), ("random", 2), ("sync", 0)):
        s = oracle_mod.OracleSim(dims, beta=beta, rule=rule, h=h, seed=seed, tie_bits=tie_bits, law=law)
        s.run_until(T, order=order, choice_seed=cs)
        st = s.stats()
        st.pop("rounds")
        out.append((s.spins().copy(), s.times().copy(), s.counters().copy(), st))
    return out


@pytest.mark.parametrize("dims", [(16, 16), (13, 7), (2, 2), (2, 5), (4, 4, 4), (2, 2, 2), (3, 2, 5)])
@pytest.mark.parametrize("tie_bits", [0, 28, 31])
def test_order_independence(oracle_mod, dims, tie_bits):
    """the trajectory is unique and independent of execution order."""
    res = _run_all_orders(oracle_mod, dims, 6.0, tie_bits, seed=1234, rule=tie_bits % 2,
                          h=0.1 if tie_bits else 0.0)
    ref = res[0]
    for other in res[1:]:
        for a, b in zip(ref[:3], other[:3]):
            assert np.array_equal(a, b)
        assert ref[3] == other[3]


@pytest.mark.parametrize("dims", [(16, 16), (2, 5), (4, 4, 4)])
@pytest.mark.parametrize("law", [1, 2, 3])
def test_order_independence_other_laws(oracle_mod, dims, law):
    """The uniqueness argument does not depend on the asynchrony law
    (PAPER.md:364-410): uniform and r^(1/8) increments give one trajectory in every order."""
    res = _run_all_orders(oracle_mod, dims, 6.0, 0, seed=77, rule=1, h=0.1, law=law)
    for other in res[1:]:
        for a, b in zip(res[0][:3], other[:3]):
            assert np.array_equal(a, b)
        assert res[0][3] == other[3]


def test_tie_stress_really_has_ties(oracle_mod):
    """With tie_bits = 31 (quantum 1/2), equal neighbouring times are common, so the
    order-independence test above exercises the (t, c) tie-break."""
    s = oracle_mod.OracleSim((16, 16), seed=1234, tie_bits=31)
    ties = 0
    for T in np.arange(0.5, 6.0, 0.5):
        s.run_until(T)
        t = s.times()
        ties += int((t == np.roll(t, 1, 0)).sum() + (t == np.roll(t, 1, 1)).sum())
    assert ties > 100


def test_tie_break_negative_control(oracle_mod):
    """The identity above is not vacuous: synchronous rounds with the bare
    t(c) <= min t(c') test (fig:s1c1pe step 2, no tie-break; tied neighbours then update
    concurrently from each other's old state) diverge from the oracle once ties exist,
    and agree with it when there are none."""
    def run(order, tie_bits):
        s = oracle_mod.OracleSim((16, 16), seed=1234, tie_bits=tie_bits, beta=0.44)
        s.run_until(6.0, order=order)
        return s.spins().copy(), s.stats()["event_hash"]
    assert run("pq", 0)[1] == run("naive_leq", 0)[1]
    a, b = run("pq", 31), run("naive_leq", 31)
    assert a[1] != b[1] and not np.array_equal(a[0], b[0])


def test_run_until_composition(oracle_mod):
    a = oracle_mod.OracleSim((20, 12), beta=0.5, seed=8)
    for T in (0.0, 0.3, 2.0, 2.0, 5.5, 9.0):
        a.run_until(T)
    b = oracle_mod.OracleSim((20, 12), beta=0.5, seed=8)
    b.run_until(9.0)
    assert np.array_equal(a.spins(), b.spins())
    assert np.array_equal(a.times(), b.times())
    assert a.stats() == b.stats()
    with pytest.raises(ValueError):
        a.run_until(1.0)


def _boltzmann(dims, beta, J, h):
    """Brute force over all 2^N states; bonds along +e_a with wrap and multiplicity
    (a side of 2 counts the same pair twice, P6)."""
    N = int(np.prod(dims))
    nd = len(dims)
    w = np.zeros(1 << N)
    idx = np.arange(N).reshape(dims[::-1])
    for code in range(1 << N):
        s = np.array([1 if (code >> c) & 1 else -1 for c in range(N)]).reshape(dims[::-1])
        B = 0
        for ax in range(nd):
            B += int((s * np.roll(s, -1, axis=nd - 1 - ax)).sum())
        M = int(s.sum())
        w[code] = math.exp(-beta * (-J * B - h * M))
    del idx
    return w / w.sum()


def _chi2_ok(counts, probs, alpha=1e-4):
    exp = probs * counts.sum()
    keep = exp >= 5
    obs = np.append(counts[keep], counts[~keep].sum())
    e = np.append(exp[keep], exp[~keep].sum())
    if e[-1] == 0:
        obs, e = obs[:-1], e[:-1]
    chi2, p = sstats.chisquare(obs, e)
    return p > alpha, p


@pytest.mark.parametrize("dims,n_rep,beta,h", [((2, 2), 20000, 0.2, 0.0), ((3, 3), 30000, 0.2, 0.0),
                                                ((2, 2, 2), 30000, 0.2, 0.0), ((2, 2), 20000, 0.44, 0.1),
                                                ((3, 3), 20000, 0.44, 0.1)])
@pytest.mark.parametrize("rule", [0, 1])
def test_stationary_distribution_is_boltzmann(oracle_mod, dims, n_rep, rule, beta, h):
    """Replicas (independent seeds) sampled at T >> the relaxation time of these lattices
    (T = 25 at beta = 0.2; T = 150 at beta = 0.44, where tunnelling between the +/- sectors
    of the 3x3 torus is slow) match the exact Boltzmann law pi ~ exp(-beta(-J B - h M))
    (SPEC.md:267, 722)."""
    T = 25.0 if beta < 0.3 else 150.0
    n_rep = n_rep if beta < 0.3 else min(n_rep, 20000)
    hist = oracle_mod.replica_hist(dims, beta, 1.0, h, rule, seed0=1000 * rule + 17, n_rep=n_rep, T=T)
    ok, p = _chi2_ok(hist.astype(float), _boltzmann(dims, beta, 1.0, h))
    assert ok, p


def test_boltzmann_negative_control(oracle_mod):
    """The chi^2 check has power: the same histogram against the law with a flipped field
    sign is rejected."""
    hist = oracle_mod.replica_hist((3, 3), 0.44, 1.0, 0.1, 0, seed0=5, n_rep=20000, T=150.0)
    ok, _ = _chi2_ok(hist.astype(float), _boltzmann((3, 3), 0.44, 1.0, -0.1))
    assert not ok


@pytest.mark.parametrize("rule", [0, 1])
def test_time_weighted_3d_2x2x2(oracle_mod, rule):
    """2x2x2 at beta = 0.44, h = 0.1: with doubled bonds the +/- sectors tunnel slowly, so a
    long single run's time-weighted occupation is compared (total variation < 0.015)."""
    w = oracle_mod.time_weighted_hist((2, 2, 2), 0.44, 1.0, 0.1, rule, seed=3, T0=50.0, T1=1.0e6)
    p = w / w.sum()
    tv = 0.5 * np.abs(p - _boltzmann((2, 2, 2), 0.44, 1.0, 0.1)).sum()
    assert tv < 0.015, tv


def test_time_weighted_low_temperature(oracle_mod):
    """beta = 1, h = 0.1 (config 5's temperature), Metropolis, 2x2: sector switches are too
    rare for the global histogram, so compare within each sector the time-weighted
    occupation of the single-flip excitations relative to the ground state with the
    Boltzmann ratio (about 2.7e-4 for the up sector; 15 % tolerance, ~5 sigma)."""
    w = oracle_mod.time_weighted_hist((2, 2), 1.0, 1.0, 0.1, 1, seed=3, T0=50.0, T1=2.0e6)
    P = _boltzmann((2, 2), 1.0, 1.0, 0.1)
    for ground in (0b1111, 0b0000):
        exc = [ground ^ (1 << c) for c in range(4)]
        got = w[exc].sum() / w[ground]
        want = P[exc].sum() / P[ground]
        assert abs(got / want - 1) < 0.15, (ground, got, want)


def onsager_u(beta):
    """Onsager's energy per spin of the square-lattice Ising model, J = 1, h = 0."""
    mpmath.mp.dps = 50
    b = mpmath.mpf(beta)
    k = 2 * mpmath.sinh(2 * b) / mpmath.cosh(2 * b) ** 2
    K = mpmath.ellipk(k ** 2)
    return float(-mpmath.coth(2 * b) * (1 + 2 / mpmath.pi * (2 * mpmath.tanh(2 * b) ** 2 - 1) * K))


def test_onsager_values():
    # textbook values of u(beta); guards the helper itself
    assert abs(onsager_u(0.3) - (-0.704499)) < 2e-5
    assert abs(onsager_u(0.6) - (-1.909086)) < 2e-5
    assert abs(onsager_u(0.44068679350977) + math.sqrt(2)) < 1e-3


@pytest.mark.slow
@pytest.mark.parametrize("beta,init_q", [(0.3, 0.5), (0.6, 0.0)])
def test_onsager_energy(oracle_mod, beta, init_q):
    """L = 128 heat-bath, burn-in T = 60, E/N averaged at integer times 60..400; batch-means
    error; |mean - u_Onsager| < 5 sigma + 0.002 (finite-size bias at L = 128 is far below)."""
    L = 128
    s = oracle_mod.OracleSim((L, L), beta=beta, seed=21, init_q=init_q)
    s.run_until(60.0)
    e = []
    for T in range(61, 401):
        s.run_until(float(T))
        e.append(-s.stats()["bond_sum"] / (L * L))
    e = np.array(e)
    nb = 17
    bm = e[: len(e) // nb * nb].reshape(nb, -1).mean(axis=1)
    sigma = bm.std(ddof=1) / math.sqrt(nb)
    u = onsager_u(beta)
    assert abs(e.mean() - u) < 5 * sigma + 0.002, (e.mean(), u, sigma)


@pytest.mark.parametrize("dims,kw,Ts", [
    ((64, 48), dict(beta=0.4406868), [3.0, 7.25]),
    ((96, 64), dict(beta=1.0, h=0.1, rule=1, init_q=0.05), [12.0]),
    ((13, 7), dict(beta=0.6, lam=2.5), [2.0, 5.0]),
    ((12, 10, 8), dict(beta=0.2216544), [4.0]),
    ((32, 32), dict(beta=0.5, tie_bits=30), [6.0]),          # forced ties: the (t, c) order inside buckets
    ((32, 32), dict(beta=0.5, tie_bits=36), [40.0]),         # ties wider than a bucket
    ((24, 24), dict(beta=0.5, law=3), [5.0]),
    ((24, 24), dict(beta=0.5, law=1, lam=0.3), [9.0]),
])
def test_calendar_queue_equals_heap(oracle_mod, dims, kw, Ts):
    """(D) the calendar-queue form of the global priority queue processes the arrivals in the
    same (t, c) order as the binary heap (A): identical spins, times, counters, flips, hash."""
    a = oracle_mod.OracleSim(dims, seed=17, **kw)
    b = oracle_mod.OracleSim(dims, seed=17, **kw)
    for T in Ts:
        a.run_until(T)
        b.run_until(T, order="calendar")
    assert np.array_equal(a.spins(), b.spins())
    assert np.array_equal(a.times(), b.times())
    assert np.array_equal(a.counters(), b.counters())
    sa, sb = a.stats(), b.stats()
    for k in ("arrivals", "flips", "event_hash", "bond_sum", "magnetisation"):
        assert sa[k] == sb[k], k
    # composition across the two queues: heap after calendar and calendar after heap
    a.run_until(Ts[-1] + 1.5, order="calendar")
    b.run_until(Ts[-1] + 1.5)
    assert np.array_equal(a.times(), b.times()) and np.array_equal(a.spins(), b.spins())
