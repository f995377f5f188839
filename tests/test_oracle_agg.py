"""Pins of the aggregated Poisson-stream oracle (fig:amcpoi; P8):
  * m = 1 is fig:a1c1pe with per-cell streams: bit-identical to the main oracle;
  * per-subarray times and counters are the subarray's own stream (state independence);
  * an independent executor that fires ready subarrays in random order reaches the same
    trajectory (uniqueness for a fixed partition);
  * the stationary distribution of a 2 x 4 torus in 2 x 2 subarrays is Boltzmann (brute force)."""
import random

import numpy as np
import pytest

import oracle as O


@pytest.mark.parametrize("dims,rule,h", [((16, 16), 0, 0.0), ((8, 6), 1, 0.1), ((2, 2), 0, 0.0), ((5, 7), 1, 0.0)])
def test_agg_m1_is_the_main_oracle(oracle_mod, dims, rule, h):
    sp, T, n, st = oracle_mod.agg_run(dims, 1, 6.0, beta=0.44, seed=9, rule=rule, h=h)
    o = oracle_mod.OracleSim(dims, beta=0.44, seed=9, rule=rule, h=h)
    o.run_until(6.0)
    assert np.array_equal(sp, o.spins())
    assert np.array_equal(T, o.times().ravel()) and np.array_equal(n, o.counters().ravel())
    so = o.stats()
    for k in ("arrivals", "flips", "event_hash", "bond_sum", "magnetisation"):
        assert st[k] == so[k], k


def _stream(seed, C, m, lam, T_end):
    """(T, n) of subarray C from its own stream (P8), without the simulation."""
    tag_e, tag_i = (0, 1) if m == 1 else (3, 4)
    inv = int(np.floor(4294967296.0 / (lam * m * m) + 0.5))
    key = (seed & 0xFFFFFFFF, seed >> 32)

    def d(w1, w2):
        q = O.nlog_q32((w1 << 32) | w2)
        return max(1, (q * inv) >> 32)
    w = O.philox((0, C, 0, tag_i), key)
    t, k = d(w[1], w[2]), 0
    while t < T_end:
        w = O.philox((k, C, 0, tag_e), key)
        t += d(w[1], w[2])
        k += 1
    return t, k


def test_agg_times_are_the_subarray_streams(oracle_mod):
    dims, m, T = (16, 8), 4, 5.0
    sp, Tt, n, st = oracle_mod.agg_run(dims, m, T, beta=0.44, seed=21)
    for C in range(len(Tt)):
        assert (int(Tt[C]), int(n[C])) == _stream(21, C, m, 1.0, O.to_q32(T))
    assert st["arrivals"] == int(n.sum())
    assert abs(st["arrivals"] - 128 * T) < 5 * np.sqrt(128 * T)


def _random_order(dims, m, T, beta, seed, rule, h, choice_seed):
    """Independent executor (pure Python over the oracle's primitives): repeatedly pick a random
    subarray whose next arrival is ready — its chosen cell's outside neighbours sit in
    subarrays with larger (T, C) — and process it."""
    nx, ny = dims
    mx, my = nx // m, ny // m
    NC = mx * my
    tag_e, tag_i = (0, 1) if m == 1 else (3, 4)
    key = (seed & 0xFFFFFFFF, seed >> 32)
    inv = int(np.floor(4294967296.0 / (m * m) + 0.5))
    thr = O.flip_table(2, beta, 1.0, h, rule)
    s = np.zeros((ny, nx), np.int64)
    for y in range(ny):
        for x in range(nx):
            s[y, x] = -1 if O.philox((0, y * nx + x, 0, 1), key)[0] < int(np.floor(0.5 * 4294967296.0)) else 1
    Tt, n = [], [0] * NC
    for C in range(NC):
        w = O.philox((0, C, 0, tag_i), key)
        Tt.append(max(1, (O.nlog_q32((w[1] << 32) | w[2]) * inv) >> 32))
    Tend = O.to_q32(T)
    rng = random.Random(choice_seed)
    while True:
        ready = []
        for C in range(NC):
            if Tt[C] >= Tend:
                continue
            w = O.philox((n[C], C, 0, tag_e), key)
            l = (w[3] * m * m) >> 32                     # P8 Step 2 (= w3 >> (32 - log2 m^2) for powers of 2)
            X, Y = C % mx, C // mx
            x, y = X * m + l % m, Y * m + l // m
            ok = True
            for xx, yy in (((x - 1) % nx, y), ((x + 1) % nx, y), (x, (y - 1) % ny), (x, (y + 1) % ny)):
                C2 = (yy // m) * mx + xx // m
                if C2 != C and not (Tt[C] < Tt[C2] or (Tt[C] == Tt[C2] and C < C2)):
                    ok = False
            if ok:
                ready.append((C, w, x, y))
        if not ready:
            break
        C, w, x, y = rng.choice(ready)
        sig = s[y, (x - 1) % nx] + s[y, (x + 1) % nx] + s[(y - 1) % ny, x] + s[(y + 1) % ny, x]
        sc = s[y, x]
        if w[0] < thr[(sig + 4) // 2 + 5 * (sc + 1) // 2]:
            s[y, x] = -sc
        Tt[C] += max(1, (O.nlog_q32((w[1] << 32) | w[2]) * inv) >> 32)
        n[C] += 1
    return s.astype(np.int8), np.array(Tt, np.uint64), np.array(n, np.uint32)


@pytest.mark.parametrize("dims,m", [((8, 8), 2), ((8, 4), 4), ((6, 6), 2), ((9, 6), 3), ((24, 12), 12)])
def test_agg_order_independence(oracle_mod, dims, m):
    sp, Tt, n, st = oracle_mod.agg_run(dims, m, 4.0, beta=0.5, seed=17, rule=1, h=0.1)
    for cs in (1, 2):
        s2, T2, n2 = _random_order(dims, m, 4.0, 0.5, 17, 1, 0.1, cs)
        assert np.array_equal(sp, s2) and np.array_equal(Tt, T2) and np.array_equal(n, n2)


def test_agg_stationary_boltzmann(oracle_mod):
    """2 x 4 torus (doubled bonds along the side of 2), 2 x 2 subarrays, heat-bath at
    beta = 0.44: replica histogram at T = 30 vs exact Boltzmann weights (chi-square)."""
    from scipy import stats
    nx, ny, beta = 4, 2, 0.44
    n_rep = 12000
    hist = np.zeros(256)
    for r in range(n_rep):
        sp, _, _, _ = oracle_mod.agg_run((nx, ny), 2, 30.0, beta=beta, seed=1000 + r)
        code = int(sum(1 << i for i, v in enumerate(sp.ravel()) if v > 0))
        hist[code] += 1
    E = np.zeros(256)
    for code in range(256):
        s = np.array([1 if (code >> i) & 1 else -1 for i in range(8)]).reshape(ny, nx)
        B = (s * (np.roll(s, -1, 1) + np.roll(s, -1, 0))).sum()
        E[code] = -B
    p = np.exp(-beta * E)
    p /= p.sum()
    chi = stats.chisquare(hist, n_rep * p)
    assert chi.pvalue > 1e-3, chi


# ---------------------------------------------------------------- modified BKL (P9)
def _boltzmann_EM(nx, ny, beta, h):
    """Exact joint distribution of (B, M) on an nx x ny torus (bonds with multiplicity)."""
    n = nx * ny
    codes = np.arange(1 << n, dtype=np.int64)
    s = np.where(((codes[:, None] >> np.arange(n)) & 1) > 0, 1, -1).reshape(-1, ny, nx)
    B = (s * (np.roll(s, -1, 2) + np.roll(s, -1, 1))).sum(axis=(1, 2))
    M = s.sum(axis=(1, 2))
    w = np.exp(beta * (B + h * M))
    return B, M, w / w.sum()


@pytest.mark.parametrize("m,rule,h,beta", [(4, 0, 0.0, 0.44), (4, 1, 0.1, 0.3), (2, 0, 0.1, 0.3)])
def test_bkl_stationary_boltzmann(oracle_mod, m, rule, h, beta):
    """4 x 4 torus: one 4 x 4 subarray (kernel 2 x 2, layer 12: both procedures active) or four
    2 x 2 subarrays (layer only, with waits). The joint (B, M) histogram of independent
    replicas at T = 40 matches exact enumeration (chi-square). (With a field at beta = 0.44 the
    4 x 4 magnetisation relaxes too slowly for T = 40: the standard model misses too.)"""
    from scipy import stats
    B, M, p = _boltzmann_EM(4, 4, beta, h)
    keys = sorted(set(zip(B.tolist(), M.tolist())))
    idx = {k: i for i, k in enumerate(keys)}
    pk = np.zeros(len(keys))
    for b, mm, pp in zip(B, M, p):
        pk[idx[(int(b), int(mm))]] += pp
    n_rep = 6000
    hist = np.zeros(len(keys))
    for r in range(n_rep):
        sp, _, _, st = oracle_mod.agg_run((4, 4), m, 40.0, beta=beta, h=h, rule=rule, seed=5000 + r, bkl=True)
        hist[idx[(int(st["bond_sum"]), int(st["magnetisation"]))]] += 1
    keep = n_rep * pk >= 5
    obs = np.append(hist[keep], hist[~keep].sum())
    exp = np.append(n_rep * pk[keep], n_rep * pk[~keep].sum())
    chi = stats.chisquare(obs, exp * obs.sum() / exp.sum())
    assert chi.pvalue > 1e-3, chi


def test_bkl_flip_rate_matches_standard_model(oracle_mod):
    """The n-fold way skips rejected attempts only: over the same time horizon the number of
    spin flips per unit time (a property of the continuous-time process) agrees with the
    standard model's (PQ oracle) within statistical error, while BKL needs fewer events."""
    dims, T, beta = (32, 32), 40.0, 0.6
    fb, eb, fs = [], [], []
    for sd in range(4):
        _, _, _, st = oracle_mod.agg_run(dims, 8, T, beta=beta, seed=100 + sd, bkl=True)
        fb.append(st["flips"]); eb.append(st["arrivals"])
        o = oracle_mod.OracleSim(dims, beta=beta, seed=200 + sd)
        o.run_until(T)
        fs.append(o.stats()["flips"])
    fb, fs = np.array(fb, float), np.array(fs, float)
    assert abs(fb.mean() - fs.mean()) < 5 * np.sqrt((fb.var() + fs.var() + fb.mean()) / 4)
    assert np.mean(eb) < 0.8 * 1024 * T           # rejections were skipped in the kernels


def _bkl_random_order(dims, m, T, beta, h, rule, seed, choice_seed):
    """Independent executor of P9 (pure Python over the oracle's primitives) that processes a
    random ready subarray at each step: its next event is ready when it is a kernel event, or a
    layer event whose outside neighbours sit in subarrays with larger (T, C)."""
    nx, ny = dims
    mx, my = nx // m, ny // m
    NC = mx * my
    key = (seed & 0xFFFFFFFF, seed >> 32)
    thr = O.flip_table(2, beta, 1.0, h, rule)
    s = np.zeros((ny, nx), np.int64)
    for y in range(ny):
        for x in range(nx):
            s[y, x] = -1 if O.philox((0, y * nx + x, 0, 1), key)[0] < 2 ** 31 else 1

    def classes(C):
        X, Y = C % mx, C // mx
        cls, W = [], 0
        for l in range(m * m):
            i, j = l % m, l // m
            if i in (0, m - 1) or j in (0, m - 1):
                cls.append(-1); W += 2 ** 32; continue
            x, y = X * m + i, Y * m + j
            sig = s[y, x - 1] + s[y, x + 1] + s[y - 1, x] + s[y + 1, x]
            k = (sig + 4) // 2 + 5 * (s[y, x] + 1) // 2
            cls.append(k); W += thr[k]
        return cls, W

    def delta(w2, w3, W):
        q = O.nlog_q32((w2 << 32) | w3)
        inv = int(np.floor(np.float64(18446744073709551616.0) / (np.float64(1.0) * np.float64(W)) + np.float64(0.5)))
        return max(1, (q * inv) >> 32)

    Tt, n = [], [0] * NC
    for C in range(NC):
        w = O.philox((0, C, 0, 6), key)
        Tt.append(delta(w[2], w[3], classes(C)[1]))
    Tend, rng = O.to_q32(T), random.Random(choice_seed)
    W0 = (4 * m - 4) << 32
    while True:
        ready = []
        for C in range(NC):
            if Tt[C] >= Tend:
                continue
            w = O.philox((n[C], C, 0, 5), key)
            cls, W = classes(C)
            u = ((((w[0] << 32) | w[1]) * W) >> 64)
            X, Y = C % mx, C // mx
            if u < W0:
                b = u >> 32
                l = [q for q in range(m * m) if cls[q] < 0][b]
                x, y = X * m + l % m, Y * m + l // m
                ok = True
                for xx, yy in (((x - 1) % nx, y), ((x + 1) % nx, y), (x, (y - 1) % ny), (x, (y + 1) % ny)):
                    C2 = (yy // m) * mx + xx // m
                    if C2 != C and not (Tt[C] < Tt[C2] or (Tt[C] == Tt[C2] and C < C2)):
                        ok = False
                if ok:
                    ready.append((C, w, u, l, True))
            else:
                o = u - W0
                for kc in range(10):
                    Wk = sum(1 for q in cls if q == kc) * thr[kc]
                    if o < Wk:
                        break
                    o -= Wk
                l = [q for q in range(m * m) if cls[q] == kc][o // thr[kc]]
                ready.append((C, w, u, l, False))
        if not ready:
            break
        C, w, u, l, layer = rng.choice(ready)
        X, Y = C % mx, C // mx
        x, y = X * m + l % m, Y * m + l // m
        if layer:
            sig = s[y, (x - 1) % nx] + s[y, (x + 1) % nx] + s[(y - 1) % ny, x] + s[(y + 1) % ny, x]
            if (u & 0xFFFFFFFF) < thr[(sig + 4) // 2 + 5 * (s[y, x] + 1) // 2]:
                s[y, x] = -s[y, x]
        else:
            s[y, x] = -s[y, x]
        Tt[C] += delta(w[2], w[3], classes(C)[1])
        n[C] += 1
    return s.astype(np.int8), np.array(Tt, np.uint64), np.array(n, np.uint32)


@pytest.mark.parametrize("dims,m", [((8, 8), 4), ((16, 8), 8), ((8, 8), 2), ((9, 6), 3), ((24, 12), 12)])
def test_bkl_order_independence(oracle_mod, dims, m):
    sp, Tt, n, st = oracle_mod.agg_run(dims, m, 3.0, beta=0.6, h=0.1, rule=1, seed=31, bkl=True)
    s2, T2, n2 = _bkl_random_order(dims, m, 3.0, 0.6, 0.1, 1, 31, 7)
    assert np.array_equal(sp, s2) and np.array_equal(Tt, T2) and np.array_equal(n, n2)
