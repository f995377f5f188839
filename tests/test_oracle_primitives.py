"""Pins of the oracle's primitives (docs/PRIMITIVES.md P1-P4, P7) against things other than
the oracle itself: published known-answer vectors, the cuRAND host library, mpmath's
logarithm/exponential, and the Appendix's worked values (SPEC.md:233-245 restating
PAPER.md:1691-1701, 1803)."""
import ctypes
import math
import os
import random

import mpmath
import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
mpmath.mp.dps = 50


def _kat_rows():
    rows = []
    with open(os.path.join(HERE, "golden", "philox4x32_10_kat.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            v = [int(x, 16) for x in line.split()]
            rows.append((tuple(v[0:4]), tuple(v[4:6]), tuple(v[6:10])))
    return rows


@pytest.mark.parametrize("ctr,key,out", _kat_rows())
def test_philox_known_answers(oracle_mod, ctr, key, out):
    assert oracle_mod.philox(ctr, key) == out


def _curand_host():
    for p in ("/usr/local/cuda/lib64/libcurand.so", "/usr/local/cuda/lib64/libcurand.so.10"):
        if os.path.exists(p):
            return ctypes.CDLL(p)
    return None


def test_philox_matches_curand_host_generator(oracle_mod):
    """cuRAND's host Philox4x32-10 generator (a library routine, independent of our code):
    block i of a stream with seed S is Philox(ctr=(0,0,i,0), key=S) (established in this
    test by the KAT-consistent block 0)."""
    cr = _curand_host()
    if cr is None:
        pytest.skip("libcurand not present")
    g = ctypes.c_void_p()
    assert cr.curandCreateGeneratorHost(ctypes.byref(g), 161) == 0  # PHILOX4_32_10
    try:
        rnd = random.Random(7)
        for seed in [0, 1, 12345, 0xFFFFFFFF, 1 << 32, 0x0123456789ABCDEF, rnd.getrandbits(64)]:
            cr.curandSetPseudoRandomGeneratorSeed(g, ctypes.c_ulonglong(seed))
            cr.curandSetGeneratorOffset(g, ctypes.c_ulonglong(0))
            nblk = 4096
            out = np.zeros(4 * nblk, np.uint32)
            assert cr.curandGenerate(g, out.ctypes.data_as(ctypes.c_void_p), out.size) == 0
            key = (seed & 0xFFFFFFFF, seed >> 32)
            for i in list(range(64)) + [rnd.randrange(nblk) for _ in range(64)]:
                assert oracle_mod.philox((0, 0, i, 0), key) == tuple(int(v) for v in out[4 * i:4 * i + 4])
    finally:
        cr.curandDestroyGenerator(g)


def _exact_nlog(X):
    x = X | 1
    return -mpmath.log(mpmath.mpf(x) / mpmath.mpf(2) ** 64) * mpmath.mpf(2) ** 32


def _nlog_inputs(n_random=20000, seed=3):
    r = random.Random(seed)
    xs = [r.getrandbits(64) for _ in range(n_random)]
    M = (1 << 64) - 1
    xs += [0, 1, 2, 3, 1 << 63, (1 << 63) + 1, M, M - 1]
    for k in range(64):
        xs += [1 << k, (1 << k) + 1, (1 << (k + 1)) - 1]
    for i in range(256):                       # every table-segment boundary, several octaves
        for sh in (0, 1, 7, 20, 40, 62):
            b = ((1 << 63) | (i << 55)) >> sh
            for d in (-(1 << 25), -1, 0, 1, 1 << 25):
                if 0 <= b + d <= M:
                    xs.append(b + d)
    return xs


def test_nlog_within_one_unit_of_mpmath(oracle_mod):
    """P3 contract |q - (-ln u) 2^32| <= 1 (the survey's proposal allowed 2)."""
    worst = 0.0
    for X in _nlog_inputs():
        err = abs(float(oracle_mod.nlog_q32(X) - _exact_nlog(X)))
        worst = max(worst, err)
    assert worst <= 1.0, worst


def test_nlog_within_one_unit_1e7(oracle_mod):
    """The P3 contract at SURVEY 8(c)'s volume: 10^7 random inputs (plus the edge set), the oracle's
    q against -ln(x / 2^64) 2^32 evaluated in x87 extended precision (64-bit mantissa: x is exact,
    the reference's absolute error is ~1e-8 units); the few inputs whose error lies within 1e-6 of
    the bound are re-checked with mpmath at 50 digits."""
    rng = np.random.default_rng(11)
    X = np.concatenate([rng.integers(0, 2 ** 63, size=10 ** 7, dtype=np.uint64) * np.uint64(2) +
                        rng.integers(0, 2, size=10 ** 7).astype(np.uint64),
                        np.array(_nlog_inputs(n_random=0), np.uint64)])
    q = oracle_mod.nlog_batch(X)
    x = (X | np.uint64(1)).astype(np.longdouble)
    ref = -np.log(x / np.longdouble(2) ** 64) * np.longdouble(2) ** 32
    err = np.abs(q.astype(np.longdouble) - ref)
    border = np.nonzero(err > 1 - 1e-6)[0]
    for i in border:
        mpmath.mp.dps = 50
        assert abs(int(q[i]) - _exact_nlog(int(X[i]))) <= 1, int(X[i])
    assert float(err.max()) <= 1 + 1e-6
    assert len(border) < 100


def test_nlog_edge_values(oracle_mod):
    assert oracle_mod.nlog_q32((1 << 64) - 1) == 0            # u -> 1: -ln u -> 0, Delta clamps to 1
    assert oracle_mod.delta(0xFFFFFFFF, 0xFFFFFFFF) == 1
    assert oracle_mod.nlog_q32((1 << 63) + 1) == 2977044472    # ln 2 * 2^32 = 2977044471.82
    assert oracle_mod.nlog_q32(0) == 190530846196              # 64 ln 2 * 2^32
    assert oracle_mod.nlog_q32(1) == 190530846196


def test_nlog_monotone(oracle_mod):
    xs = sorted(set(X | 1 for X in _nlog_inputs(5000, 11)))
    qs = [oracle_mod.nlog_q32(X) for X in xs]
    assert all(a >= b for a, b in zip(qs, qs[1:]))


def test_increment_is_exponential(oracle_mod):
    """Eq. newt1i with Philox draws: Delta/2^32 ~ Exp(lambda). KS + mean."""
    from scipy import stats
    for lam in (1.0, 2.5):
        d = []
        for c in range(20000):
            w = oracle_mod.philox((0, c, 0, 0), (99, 7))
            d.append(oracle_mod.delta(w[1], w[2], lam) / 2.0 ** 32)
        d = np.array(d)
        ks = stats.kstest(d, "expon", args=(0, 1 / lam))
        assert ks.pvalue > 1e-4, ks
        assert abs(d.mean() - 1 / lam) < 4 * (1 / lam) / math.sqrt(len(d))


def test_increment_lambda_scaling(oracle_mod):
    """Delta(lambda) = floor(q * round(2^32/lambda) / 2^32): for lambda = 1 it is q itself."""
    r = random.Random(5)
    for _ in range(2000):
        w1, w2 = r.getrandbits(32), r.getrandbits(32)
        q = oracle_mod.nlog_q32((w1 << 32) | w2)
        assert oracle_mod.delta(w1, w2, 1.0) == max(1, q)
        assert abs(oracle_mod.delta(w1, w2, 4.0) - q / 4) <= 1
        assert abs(oracle_mod.delta(w1, w2, 0.5) - 2 * q) <= 1


def test_tie_quantisation(oracle_mod):
    r = random.Random(9)
    for k in (8, 28, 31):
        for _ in range(500):
            w1, w2 = r.getrandbits(32), r.getrandbits(32)
            d = oracle_mod.delta(w1, w2, 1.0, k)
            assert d % (1 << k) == 0 and d >= (1 << k)


def _p_exact(s, sigma, beta, J, h, rule):
    dE = 2 * (J * s * sigma + h * s)
    if rule == 0:
        x = mpmath.e ** (-beta * dE)
        return x / (1 + x)
    return min(mpmath.mpf(1), mpmath.e ** (-beta * dE))


@pytest.mark.parametrize("ndim", [2, 3])
@pytest.mark.parametrize("rule", [0, 1])
@pytest.mark.parametrize("beta,J,h", [(0.4406868, 1, 0), (1.0, 1, 0.1), (0.2216544, 1, 0),
                                      (0.0, 1, 0), (3.0, 0.5, -0.7), (400.0, 1, 0)])
def test_flip_table_against_formula(oracle_mod, ndim, rule, beta, J, h):
    """P4 via mpmath: thr = floor(p 2^32) within one unit; index layout of PAPER.md:1803."""
    thr = oracle_mod.flip_table(ndim, beta, J, h, rule)
    z = 2 * ndim
    assert len(thr) == 2 * (z + 1)
    for s in (-1, 1):
        for sigma in range(-z, z + 1, 2):
            idx = (sigma + z) // 2 + (z + 1) * (s + 1) // 2
            p = _p_exact(s, sigma, beta, J, h, rule)
            assert abs(thr[idx] - p * 2 ** 32) <= 1.0 + 1e-6, (s, sigma, thr[idx], p)
            assert 0 <= thr[idx] <= 2 ** 32


def test_flip_table_appendix_values(oracle_mod):
    """J=1, H=0, T=1 (Appendix; values restated in SPEC.md:233-236):
    s=+1: Sigma=+4 -> 3.3535e-4, Sigma=0 -> 1/2, Sigma=-4 -> 0.99966; index examples
    (SPEC.md:242-245): (-1,-4)->0, (+1,+4)->9, (+1,0)->7."""
    thr = oracle_mod.flip_table(2, 1.0, 1.0, 0.0, 0)
    assert abs(thr[9] / 2 ** 32 - 3.3535e-4) < 5e-8
    assert thr[7] == 2 ** 31
    assert abs(thr[5] / 2 ** 32 - 0.99966) < 5e-6
    # s=-1, Sigma=-4: the -1 spin is aligned with its neighbours -> same as (+1, +4)
    assert thr[0] == thr[9]
    # beta = 0: heat-bath 1/2, Metropolis always
    assert set(oracle_mod.flip_table(2, 0.0, 1.0, 0.3, 0)) == {2 ** 31}
    assert set(oracle_mod.flip_table(3, 0.0, 1.0, 0.3, 1)) == {2 ** 32}


def test_event_hash_term(oracle_mod):
    """P7 term h = (w3 | 1) (t ^ (l << 1) ^ s') mod 2^64 (docs/PRIMITIVES.md; a checksum of
    our own design): the C implementation against big-int arithmetic on extreme and random
    words, and injectivity in t for a fixed draw (odd multiplier), so two arrivals of one draw
    at different times never cancel."""
    M = (1 << 64) - 1
    r = random.Random(7)
    cases = [(0, 0, 0, -1), (0xFFFFFFFF, M, 0, 1), (1, 1 << 63, 63, 1), (0xFFFFFFFE, 12345, 0, -1)]
    cases += [(r.getrandbits(32), r.getrandbits(64), r.randrange(64), r.choice((-1, 1))) for _ in range(2000)]
    for w3, t, l, s in cases:
        assert oracle_mod.ev_hash(w3, t, l, s) == ((w3 | 1) * (t ^ (l << 1) ^ (1 if s > 0 else 0))) & M
    w3 = r.getrandbits(32)
    ts = [r.getrandbits(40) for _ in range(3000)]
    assert len({oracle_mod.ev_hash(w3, t, 0, 1) for t in ts}) == len(set(ts))


def test_event_hash_of_the_first_arrival(oracle_mod):
    """The oracle's event_hash after exactly one arrival equals the P7 term built from that
    arrival's own P1 draw (w3 of Philox(seed; ctr = (0, c, 0, 0))), its time and new spin."""
    dims, seed = (6, 5), 0x1234_5678_9ABC
    o = oracle_mod.OracleSim(dims, beta=0.44, seed=seed)
    t0 = o.times().ravel()
    c = int(np.lexsort((np.arange(t0.size), t0))[0])     # smallest (t, c)
    o.run_until_q32(int(t0[c]) + 1)
    st = o.stats()
    assert st["arrivals"] == 1
    w = oracle_mod.philox((0, c, 0, 0), (seed & 0xFFFFFFFF, seed >> 32))
    assert st["event_hash"] == oracle_mod.ev_hash(w[3], int(t0[c]), 0, int(o.spins().ravel()[c]))


# ---------------------------------------------------------------- P3L asynchrony laws
def test_law_uniform_is_the_raw_word(oracle_mod):
    """Law 1, next_t - t uniform on (0,1): U = w1, i.e. (w1/2^32) is the
    uniform variate; the increment is U/lambda clamped to >= 1 unit."""
    r = random.Random(21)
    for _ in range(2000):
        w1, w2 = r.getrandbits(32), r.getrandbits(32)
        assert oracle_mod.law_q32(w1, w2, 1) == w1
        assert oracle_mod.delta(w1, w2, 1.0, 0, 1) == max(1, w1)
        assert abs(oracle_mod.delta(w1, w2, 2.0, 0, 1) - w1 / 2) <= 1
    assert oracle_mod.delta(0, 5, 1.0, 0, 1) == 1


def test_law_root8_within_one_unit_of_mpmath(oracle_mod):
    """Law 2, next_t - t = r^(1/8): U = floor(r^(1/8) 2^32) with
    r = (w1 + 1/2) 2^-32, within one unit of the exact real value; monotone in w1."""
    r = random.Random(22)
    ws = [0, 1, 2, 3, 255, 256, 2 ** 31, 2 ** 32 - 2, 2 ** 32 - 1] + [r.getrandbits(32) for _ in range(4000)]
    for w1 in ws:
        exact = mpmath.floor(mpmath.root((mpmath.mpf(w1) + mpmath.mpf(0.5)) / 2 ** 32, 8) * 2 ** 32)
        assert abs(int(oracle_mod.law_q32(w1, 0, 2)) - int(exact)) <= 1, w1
    ws = sorted(set(ws))
    us = [oracle_mod.law_q32(w, 0, 2) for w in ws]
    assert all(a <= b for a, b in zip(us, us[1:]))
    assert oracle_mod.law_q32(2 ** 32 - 1, 0, 2) == 2 ** 32 - 1     # r^(1/8) < 1 always


def test_law_root8_distribution(oracle_mod):
    """(U/2^32)^8 of Philox draws is Uniform(0,1) (KS); mean of U/2^32 is 8/9."""
    from scipy import stats
    v = []
    for c in range(20000):
        w = oracle_mod.philox((0, c, 0, 0), (41, 3))
        v.append(oracle_mod.law_q32(w[1], w[2], 2) / 2.0 ** 32)
    v = np.array(v)
    assert stats.kstest(v ** 8, "uniform").pvalue > 1e-4
    assert abs(v.mean() - 8 / 9) < 4 * math.sqrt(8 / 10 - (8 / 9) ** 2) / math.sqrt(len(v))


@pytest.mark.parametrize("law", [1, 2, 3])
def test_law_closed_form_times(oracle_mod, law):
    """Arrival times are state-independent under every law: the oracle's
    final (t, n) equal each cell's own partial sums."""
    o = oracle_mod.OracleSim((12, 10), beta=0.44, seed=5, law=law)
    o.run_until(7.0)
    t, n = o.times(), o.counters()
    for c in range(120):
        tc, nc = oracle_mod.cell_time_counter(5, c, 7.0, law=law)
        assert (int(t.flat[c]), int(n.flat[c])) == (tc, nc)


def test_gauss_quantile_within_one_unit_of_mpmath(oracle_mod):
    """P3L law 3: U = floor(2^32 (1 + Phi^{-1}((w + 1/2) 2^-32) / 4)) within one unit of mpmath's exact
    value on random words, both tails (w near 0 and 2^32 - 1, |z| up to 6.3) and the centre; the
    quantile itself is odd about w = 2^31 - 1/2."""
    mpmath.mp.dps = 30
    rnd = random.Random(21)
    ws = [rnd.getrandbits(32) for _ in range(20000)]
    ws += list(range(0, 64)) + [2 ** 32 - 1 - k for k in range(64)] + [2 ** 31 + d for d in range(-64, 64)]
    ws += [rnd.getrandbits(12) for _ in range(500)] + [2 ** 32 - 1 - rnd.getrandbits(12) for _ in range(500)]
    worst = 0
    for w in ws:
        p = (mpmath.mpf(w) + mpmath.mpf(1) / 2) / 2 ** 32
        z = mpmath.sqrt(2) * mpmath.erfinv(2 * p - 1)
        x = (1 + z / 4) * 2 ** 32
        if x >= 1:
            worst = max(worst, abs(oracle_mod.gauss_u(w, w, 0, 9) - int(mpmath.floor(x))))
        assert oracle_mod.gauss_z(w) == -oracle_mod.gauss_z(2 ** 32 - 1 - w)
    assert worst <= 1, worst


def test_law_gauss_distribution(oracle_mod):
    """Law 3 (Gaussian period, the liberal reading): U / 2^32 ~ N(1, 1/4^2)
    (the rare periods below one unit are redrawn, P(z < -4) = 3e-5): mean, sd and a KS test against
    the normal CDF."""
    from scipy import stats
    v = []
    for c in range(20000):
        w = oracle_mod.philox((0, c, 0, 0), (77, 1))
        v.append(oracle_mod.law_q32(w[1], w[2], 3) / 2.0 ** 32)
    v = np.array(v)
    assert abs(v.mean() - 1.0) < 4 * 0.25 / math.sqrt(len(v))
    assert abs(v.std() - 0.25) < 0.01
    ks = stats.kstest(v, stats.norm(loc=1.0, scale=0.25).cdf)
    assert ks.pvalue > 1e-4, ks
    assert v.min() > 0


def test_law_gauss_redraws_nonpositive_periods(oracle_mod):
    """A period below one unit is never used: the words whose quantile gives 1 + z/4 <= 0
    (z <= -4, w below ~2^32 3.2e-5) are redrawn from the keyed sub-draws, deterministically."""
    lo = [w for w in range(0, 200000, 997) if 1 + oracle_mod.gauss_z(w) / 4 <= 0]
    assert lo, "expected words in the z <= -4 tail"
    for w in lo[:50]:
        u = oracle_mod.gauss_u(w, w, 77, 9)
        assert u >= 1 and u == oracle_mod.gauss_u(w, w, 77, 9) and u != oracle_mod.gauss_u(w, w, 78, 9)


def test_law4_fixed_period_per_cell(oracle_mod):
    """Law 4 (the strict reading: sigma_c = 0, m_c Gaussian): every increment of a
    cell is its fixed period, so its closed form is an arithmetic progression: t = (n + 1) P_c,
    n = the number of periods below T; the periods are N(1, 1/4^2) across cells."""
    from scipy import stats
    T = 7.0
    Tq = oracle_mod.to_q32(T)
    P = []
    for c in range(3000):
        pc = oracle_mod.cell_period_q32(5, c)
        t, n = oracle_mod.cell_time_counter(5, c, T, law=4)
        assert t == (n + 1) * pc and n * pc < Tq <= t
        P.append(pc / 2.0 ** 32)
    assert stats.kstest(np.array(P), stats.norm(loc=1.0, scale=0.25).cdf).pvalue > 1e-4


def test_law_gauss_is_a_function_of_the_draw(oracle_mod):
    """The sub-draws are keyed by (w1, w2) only: the same arrival draw gives the same period, a
    different one (almost surely) a different period."""
    a = oracle_mod.law_q32(123, 456, 3)
    assert a == oracle_mod.law_q32(123, 456, 3) and a != oracle_mod.law_q32(124, 456, 3)
    assert oracle_mod.delta(123, 456, 2.0, 0, 3) in (a // 2, a // 2 + 1, max(1, a // 2))
