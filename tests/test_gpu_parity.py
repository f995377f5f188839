"""GPU parity: the CUDA path through the C ABI against the serial oracle, element by element
(bit-exact: spins, every t(c), every n(c), and the integer statistics B, M, arrivals,
flips, P7 event hash). Sizes span several tiles and ragged tails; edge cases: 2x2 (doubled
neighbours), forced ties (P3b), run_until composition, every tile shape / rounds-per-launch /
virtual shard count (the trajectory is invariant)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

STAT_KEYS = ("arrivals", "flips", "event_hash", "bond_sum", "magnetisation", "t_min", "t_max")


@pytest.fixture(scope="module")
def aca():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_cs_0502039_b200 as aca
    return aca


def run_pair(aca, oracle_mod, dims, Ts, beta=0.4406868, J=1.0, h=0.0, lam=1.0, rule=0, seed=1,
             init_q=0.5, tie_bits=0, law=0, **opts):
    g = aca.Sim(dims, lam=lam, beta=beta, J=J, h=h, rule=rule, seed=seed, init_q=init_q, tie_bits=tie_bits, law=law,
                **opts)
    o = oracle_mod.OracleSim(dims, lam=lam, beta=beta, J=J, h=h, rule=rule, seed=seed, init_q=init_q,
                             tie_bits=tie_bits, law=law)
    assert g.flip_table() == oracle_mod.flip_table(len(dims), beta, J, h, rule)
    for T in Ts:
        g.run_until(T)
        o.run_until(T)
    return g, o


def assert_same(g, o):
    gs, gt, gn = g.spins(), g.times(), g.counters()
    os_, ot, on = o.spins(), o.times(), o.counters()
    bad_s = np.argwhere(gs != os_)
    assert bad_s.size == 0, ("spins differ at", bad_s[:5])
    assert np.array_equal(gt, ot), ("times differ at", np.argwhere(gt != ot)[:5])
    assert np.array_equal(gn, on), ("counters differ at", np.argwhere(gn != on)[:5])
    sg, so = g.stats(), o.stats()
    for k in STAT_KEYS:
        assert sg[k] == so[k], (k, sg[k], so[k])
    assert sg["cells_fired"] == so["arrivals"]


def test_philox_matches_curand_device_and_oracle(aca, oracle_mod):
    rng = np.random.default_rng(1)
    n = 1 << 20
    ctr = rng.integers(0, 2 ** 32, size=(n, 4), dtype=np.uint64).astype(np.uint32)
    key = rng.integers(0, 2 ** 32, size=(n, 2), dtype=np.uint64).astype(np.uint32)
    ctr[:16] = [[0, 0, 0, 0], [0xFFFFFFFF] * 4] * 8
    key[:16] = [[0, 0], [0xFFFFFFFF] * 2] * 8
    out, ref = aca.aca_selftest_philox(ctr, key)
    assert np.array_equal(out, ref)
    for i in list(range(16)) + list(rng.integers(0, n, 2000)):
        assert tuple(int(v) for v in out[i]) == oracle_mod.philox(tuple(int(v) for v in ctr[i]),
                                                                  tuple(int(v) for v in key[i]))


def test_nlog_bit_identical_to_oracle(aca, oracle_mod):
    rng = np.random.default_rng(2)
    X = rng.integers(0, 2 ** 63, size=1 << 20, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, 1 << 20).astype(np.uint64)
    edges = [0, 1, 2, 3, 2 ** 63, 2 ** 63 + 1, 2 ** 64 - 1, 2 ** 64 - 2] + [2 ** k for k in range(64)]
    edges += [2 ** 32 - 1, 2 ** 32 + 1, 2 ** 33 - 1, 2 ** 31 + 12345, (2 ** 32 - 1) << 32, (2 ** 32 + 7) << 30]
    edges += [(2 ** k) - 1 for k in range(2, 64)] + [(2 ** k) + 1 for k in range(1, 64)]
    for i in range(256):
        edges += [((1 << 63) | (i << 55)) >> s for s in (0, 5, 33, 62)]
    X = np.concatenate([np.array(edges, np.uint64), X])
    q, d = aca.aca_selftest_nlog(X)
    assert np.array_equal(q, oracle_mod.nlog_batch(X))
    for lam, tb in ((1.0, 0), (2.5, 0), (0.3, 0), (1.0, 28)):
        q, d = aca.aca_selftest_nlog(X[:5000], lam, tb)
        want = [oracle_mod.delta(int(x) >> 32, int(x) & 0xFFFFFFFF, lam, tb) for x in X[:5000]]
        assert list(d) == want


def test_nlog_bit_identical_1e8(aca, oracle_mod):
    """SURVEY 8(c)'s volume: the device's NLOG-2 (the shared-memory table view the tile kernels use,
    checked against the interleaved view inside the self-test) equals the oracle's on 10^8 random
    inputs, in chunks of 10^7."""
    rng = np.random.default_rng(12)
    for _ in range(10):
        X = rng.integers(0, 2 ** 63, size=10 ** 7, dtype=np.uint64) * np.uint64(2) + \
            rng.integers(0, 2, size=10 ** 7).astype(np.uint64)
        q, d = aca.aca_selftest_nlog(X)
        assert np.array_equal(q, oracle_mod.nlog_batch(X))


@pytest.mark.parametrize("law", [0, 1, 2, 3, 4])
def test_law_bit_identical_to_oracle(aca, oracle_mod, law):
    """P3L asynchrony laws: the device's unscaled increment and
    Delta equal the oracle's on random and edge inputs, for several lambda / tie settings."""
    rng = np.random.default_rng(5 + law)
    X = rng.integers(0, 2 ** 63, size=1 << 18, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, 1 << 18).astype(np.uint64)
    edges = [0, 1, 2 ** 32 - 1, 2 ** 32, 2 ** 63, 2 ** 64 - 1, 2 ** 64 - 2 ** 32] + [(2 ** k) << 32 for k in range(32)]
    X = np.concatenate([np.array(edges, np.uint64), X])
    for lam, tb in ((1.0, 0), (2.5, 0), (0.3, 0), (1.0, 28)):
        u, d = aca.aca_selftest_law(X[:20000], law, lam, tb)
        if law == 4:   # the period of law 4 from (w3, c_lo): gauss_u(w3, w3, c_lo, 10)
            want_u = [oracle_mod.gauss_u(int(x) >> 32, int(x) >> 32, int(x) & 0xFFFFFFFF, 10) for x in X[:20000]]
            assert list(u) == want_u
            continue
        want_u = [oracle_mod.law_q32(int(x) >> 32, int(x) & 0xFFFFFFFF, law) for x in X[:20000]]
        want_d = [oracle_mod.delta(int(x) >> 32, int(x) & 0xFFFFFFFF, lam, tb, law) for x in X[:20000]]
        assert list(u) == want_u
        assert list(d) == want_d


@pytest.mark.parametrize("law", [1, 2, 3, 4])
def test_law_trajectories(aca, oracle_mod, law):
    """Whole trajectories under the uniform and r^(1/8) laws: whole-lattice, tiled 2-D with
    ragged tiles, 3-D tiles, with field and both rules."""
    for dims, kw in (((6, 5), dict(rule=0)), ((200, 150), dict(rule=1, h=0.1, whole_lattice=-1)),
                     ((24, 16, 12), dict(rule=0, beta=0.22, whole_lattice=-1, tile=(8, 8, 8)))):
        g, o = run_pair(aca, oracle_mod, dims, [3.0, 6.0], seed=23, law=law, **kw)
        assert_same(g, o)


@pytest.mark.parametrize("dims", [(2, 2), (3, 3), (5, 7), (2, 5), (16, 16), (13, 7)])
@pytest.mark.parametrize("rule", [0, 1])
def test_small_whole_lattice(aca, oracle_mod, dims, rule):
    g, o = run_pair(aca, oracle_mod, dims, [3.0, 10.0], beta=0.44, rule=rule, h=0.1 * rule, seed=7)
    assert_same(g, o)


@pytest.mark.parametrize("dims", [(2, 2, 2), (4, 4, 4), (3, 2, 5), (8, 8, 8)])
def test_small_whole_lattice_3d(aca, oracle_mod, dims):
    g, o = run_pair(aca, oracle_mod, dims, [5.0], beta=0.2216544, seed=3)
    assert_same(g, o)


@pytest.mark.parametrize("sync", [0, 1])
def test_config1_exact(aca, oracle_mod, sync):
    """Config 1: 64x64 heat-bath at beta_c, T = 10, one CTA (one cell per PE rule)."""
    g, o = run_pair(aca, oracle_mod, (64, 64), [10.0], beta=0.4406868, seed=1, sync_rounds=sync)
    assert_same(g, o)
    st = g.stats()
    assert st["launches"] == 1            # whole run_until in one launch
    assert abs(st["arrivals"] - 40960) < 5 * 202


@pytest.mark.parametrize("tile", [(64, 64), (32, 32), (64, 32)])
def test_tiled_2d_ragged(aca, oracle_mod, tile):
    """Several tiles plus ragged tails in x and y."""
    g, o = run_pair(aca, oracle_mod, (200, 150), [2.0, 6.0], beta=0.40, rule=1, seed=11, tile=tile,
                    whole_lattice=-1)
    assert_same(g, o)


@pytest.mark.parametrize("max_ctas", [0, 1, 3, 7])
def test_buffer_ring_and_grid_cap(aca, oracle_mod, max_ctas):
    """The persistent grouped kernel with its grid capped (max_ctas): every CTA cycles many
    tiles through its NBUF-buffer ring, so the buffer reuse, the mbarrier parity flips and the
    prefetch issued at write-back are all exercised; 2-D (full + ragged tiles, odd width) and
    3-D, identical trajectories."""
    for dims, tile, T in (((256, 192), (64, 64), 5.0), ((200, 150), (64, 32), 4.0), ((130, 70), (32, 32), 4.0),
                          ((64, 48, 40), (32, 16, 8), 3.0), ((40, 24, 20), (16, 16, 16), 3.0)):
        beta = 0.2216544 if len(dims) == 3 else 0.4406868
        g, o = run_pair(aca, oracle_mod, dims, [T], beta=beta, seed=37, tile=tile, whole_lattice=-1, max_ctas=max_ctas)
        assert_same(g, o)


@pytest.mark.parametrize("lag,kw", [(16.0, {}), (1.0, {}), (0.3, {}), (0.05, {}), (1.0, dict(max_ctas=3)),
                                    (0.3, dict(checkerboard=-1)), (0.5, dict(lam=2.5)), (0.3, dict(tie_bits=30)),
                                    (0.3, dict(dims=(48, 32, 40), beta=0.2216544)),
                                    (0.3, dict(beta=1.0, h=0.1, rule=1, init_q=0.05, early_reject=1)),
                                    (0.3, dict(shards=4, dims=(256, 256)))])
def test_lag_window_exact(aca, oracle_mod, lag, kw):
    """The bounded-lag window on the main path (aca_options.lag): a launch
    fires only below min(T, t_min + lag), a scheduling bound, so the trajectory is the oracle's
    for every lag (checkerboard and Jacobi launches, grid cap, lambda != 1, forced ties, 3-D,
    a10, virtual shards)."""
    kw = dict(kw)
    dims = kw.pop("dims", (256, 192))
    beta = kw.pop("beta", 0.4406868)
    g, o = run_pair(aca, oracle_mod, dims, [2.0, 5.0], beta=beta, seed=77, whole_lattice=-1, lag=lag, **kw)
    assert_same(g, o)


def test_lag_window_bounds_the_spread(aca, oracle_mod, monkeypatch):
    """With a lag window the sweeps needed grow as the bound tightens (the efficiency loss of
    fig:perfbl on the real algorithm), and the result does not change. All on the grouped tile
    kernel (the resident kernel, which runs lag-free runs of this lattice, has another schedule)."""
    monkeypatch.setenv("ACA_NO_RES", "1")
    sweeps = []
    for lag in (0.0, 4.0, 1.0, 0.3):
        g = aca.Sim((512, 512), beta=0.4406868, seed=3, lag=lag)
        g.run_until(6.0)
        st = g.stats()
        sweeps.append(st["launches"])
        if lag == 0.0:
            ref = (g.spins().copy(), g.times().copy())
        else:
            assert np.array_equal(g.spins(), ref[0]) and np.array_equal(g.times(), ref[1])
    assert sweeps[0] <= sweeps[1] <= sweeps[2] < sweeps[3], sweeps


@pytest.mark.parametrize("case", ["jacobi", "jacobi_ties", "odd_tiles", "ties_cap", "rounds1_ties", "T_frac"])
def test_staging_paths(aca, oracle_mod, case):
    """Staging paths of the grouped kernel: one launch over all tiles (checkerboard -1: every
    halo word is read by threads with relaxed loads, neighbours run concurrently), odd tile
    counts (same-colour wrap neighbours: the wrapped halo by threads), forced ties with a
    capped grid, R = 1 (every round exact), and a horizon whose Q32 value has a non-zero low
    half (the T bucket tie)."""
    kw = dict(dims=(256, 192), Ts=[3.0, 6.0], seed=29, whole_lattice=-1)
    if case == "jacobi":
        kw.update(checkerboard=-1)
    elif case == "jacobi_ties":
        kw.update(checkerboard=-1, tie_bits=30)
    elif case == "odd_tiles":
        kw.update(dims=(320, 192))          # 5 x 3 tiles of 64: odd in x and y
    elif case == "ties_cap":
        kw.update(tie_bits=29, max_ctas=2)
    elif case == "rounds1_ties":
        kw.update(tie_bits=30, rounds_per_launch=1)
    elif case == "T_frac":
        kw.update(Ts=[2.3, 5.123456789])
    dims, Ts = kw.pop("dims"), kw.pop("Ts")
    g, o = run_pair(aca, oracle_mod, dims, Ts, **kw)
    assert_same(g, o)


@pytest.mark.parametrize("case", ["c5", "hb", "3d", "ties", "bulk"])
def test_early_rejection_exact(aca, oracle_mod, case, monkeypatch):
    """a10: committing arrivals that are rejected in every consistent world (and, with bulk,
    several arrivals of one cell per step) leaves the trajectory bit-identical."""
    if case == "bulk":
        monkeypatch.setenv("ACA_BULK", "8")
    kw = dict(c5=dict(dims=(256, 192), T=[20.0], beta=1.0, h=0.1, rule=1, init_q=0.05),
              hb=dict(dims=(192, 128), T=[6.0], beta=0.6, h=0.05, rule=0),
              bulk=dict(dims=(192, 128), T=[6.0], beta=0.4406868, rule=0),
              ties=dict(dims=(128, 96), T=[8.0], beta=1.0, h=0.1, rule=1, init_q=0.05, tie_bits=30),
              **{"3d": dict(dims=(48, 32, 24), T=[4.0], beta=0.5, h=0.1, rule=1, init_q=0.05)})[case]
    dims, Ts = kw.pop("dims"), kw.pop("T")
    g, o = run_pair(aca, oracle_mod, dims, Ts, seed=43, whole_lattice=-1, early_reject=1, **kw)
    assert_same(g, o)


@pytest.mark.parametrize("rounds", [1, 3, 8, 64])
def test_rounds_per_launch_invariance(aca, oracle_mod, rounds):
    g, o = run_pair(aca, oracle_mod, (256, 192), [5.0], seed=5, rounds_per_launch=rounds, whole_lattice=-1)
    assert_same(g, o)


def test_sync_rounds_tiled(aca, oracle_mod):
    g, o = run_pair(aca, oracle_mod, (192, 128), [4.0], seed=9, sync_rounds=1, whole_lattice=-1)
    assert_same(g, o)


@pytest.mark.parametrize("tile", [(32, 16, 8), (16, 16, 16), (8, 8, 8)])
def test_tiled_3d_ragged(aca, oracle_mod, tile):
    g, o = run_pair(aca, oracle_mod, (40, 24, 20), [3.0], beta=0.2216544, seed=13, tile=tile, whole_lattice=-1)
    assert_same(g, o)


@pytest.mark.parametrize("tie_bits", [28, 31])
def test_forced_ties(aca, oracle_mod, tie_bits):
    g, o = run_pair(aca, oracle_mod, (128, 96), [6.0], beta=0.44, seed=17, tie_bits=tie_bits, whole_lattice=-1)
    assert_same(g, o)
    g, o = run_pair(aca, oracle_mod, (6, 5), [6.0], beta=0.44, seed=17, tie_bits=tie_bits)
    assert_same(g, o)
    g, o = run_pair(aca, oracle_mod, (12, 10, 8), [4.0], beta=0.22, seed=17, tie_bits=tie_bits, whole_lattice=-1,
                    tile=(8, 8, 8))
    assert_same(g, o)


@pytest.mark.parametrize("halo_mode", [0, 1])
@pytest.mark.parametrize("shards", [2, 4, 8])
def test_virtual_shards(aca, oracle_mod, shards, halo_mode):
    """G row strips (2-D) / z slabs (3-D) on one device: the multi-GPU partition and halo logic.
    halo_mode 0: the tile kernels push their boundary rows into the neighbour shard's halo as
    they write back (no exchange step); 1: halo rows copied before every launch. Also an odd
    width (unvectorised write-back path) and ragged tiles."""
    g, o = run_pair(aca, oracle_mod, (128, 64 * shards // 2), [4.0], seed=19, shards=shards, halo_mode=halo_mode)
    assert_same(g, o)
    g, o = run_pair(aca, oracle_mod, (32, 16, 8 * shards), [3.0], beta=0.22, seed=19, shards=shards,
                    tile=(16, 16, 16), halo_mode=halo_mode)
    assert_same(g, o)
    g, o = run_pair(aca, oracle_mod, (77, 12 * shards), [3.0], rule=1, h=0.1, seed=29, shards=shards,
                    tile=(32, 32), halo_mode=halo_mode)
    assert_same(g, o)


def test_run_until_composition(aca, oracle_mod):
    g, o = run_pair(aca, oracle_mod, (160, 96), [0.0, 0.5, 2.0, 2.0, 7.25], seed=23, whole_lattice=-1)
    assert_same(g, o)
    g2, _ = run_pair(aca, oracle_mod, (160, 96), [7.25], seed=23, whole_lattice=-1)
    assert np.array_equal(g.spins(), g2.spins()) and g.stats()["event_hash"] == g2.stats()["event_hash"]
    import paper_cs_0502039_b200 as pkg
    with pytest.raises(pkg.AcaError):
        g.run_until(1.0)


def test_lambda_and_field(aca, oracle_mod):
    g, o = run_pair(aca, oracle_mod, (96, 80), [1.5, 3.0], lam=2.5, beta=0.7, h=-0.3, J=0.8, rule=0, seed=29,
                    whole_lattice=-1)
    assert_same(g, o)


def test_init_minority(aca, oracle_mod):
    """Config 5's initial state (all +1 but an i.i.d. 5 %) at beta = 1, h = 0.1 Metropolis."""
    g, o = run_pair(aca, oracle_mod, (256, 128), [10.0], beta=1.0, h=0.1, rule=1, init_q=0.05, seed=31,
                    whole_lattice=-1)
    assert_same(g, o)


def test_set_state_roundtrip(aca, oracle_mod):
    g = aca.Sim((64, 48), beta=0.5, seed=3, whole_lattice=-1)
    g.run_until(2.0)
    s, t, n = g.spins().copy(), g.times().copy(), g.counters().copy()
    g2 = aca.Sim((64, 48), beta=0.5, seed=3, whole_lattice=-1)
    g2.set_state(s, t, n)
    g.run_until(5.0)
    g2.run_until(5.0)
    assert np.array_equal(g.spins(), g2.spins()) and np.array_equal(g.times(), g2.times())


def test_set_state_beyond_horizon(aca, oracle_mod):
    """A restored state whose times lie far beyond the next horizon: the packed layout must keep
    every stored time (no silent loss of high time bits when the counter field grows)."""
    g, o = run_pair(aca, oracle_mod, (64, 48), [3.0], beta=0.5, seed=47, whole_lattice=-1)
    s, t, n = g.spins().copy(), g.times().copy(), g.counters().copy()
    t2 = t + np.uint64(900 << 32)           # every pending arrival 900 time units later
    g.set_state(s, t2, n)
    g.run_until(5.0)                         # nothing is below T: no arrival may fire
    assert np.array_equal(g.times(), t2) and np.array_equal(g.counters(), n) and np.array_equal(g.spins(), s)
    assert g.stats()["t_min"] == int(t2.min())
    g.run_until(904.0)
    g2 = aca.Sim((64, 48), beta=0.5, seed=47, whole_lattice=-1)   # the same state run straight to 904
    g2.set_state(s, t2, n)
    g2.run_until(904.0)
    assert np.array_equal(g.spins(), g2.spins()) and np.array_equal(g.times(), g2.times())
    assert np.array_equal(g.counters(), g2.counters()) and int(g.counters().sum() - n.sum()) > 0


def test_packed_layout_repack(aca, oracle_mod):
    """The (t, n) split of the packed word follows T: long horizons move bits from the counter
    to the time field (repack in place) and the trajectory is unchanged."""
    g, o = run_pair(aca, oracle_mod, (40, 24), [0.5, 40.0, 700.0], beta=0.44, seed=41, whole_lattice=-1,
                    tile=(32, 32))
    assert_same(g, o)
    g, o = run_pair(aca, oracle_mod, (6, 7), [3.0, 1500.0], beta=0.3, seed=41)   # whole-lattice kernel
    assert_same(g, o)


def test_counter_overflow_is_reported(aca, oracle_mod):
    """A counter that would overflow its packed field stops the run with ACA_ERANGE instead
    of wrapping."""
    import paper_cs_0502039_b200 as pkg
    g = aca.Sim((8, 8), beta=0.4, seed=3, whole_lattice=-1, tile=(32, 32))
    s, t, n = g.spins().copy(), g.times().copy(), g.counters().copy()
    g.set_state(s, t, n)
    nb = g.stats()["counter_bits"]
    assert nb >= 9
    n[:] = 2 ** nb - 2          # one more event fills the field, the next would overflow
    g.set_state(s, t, n)
    assert g.stats()["counter_bits"] == nb
    with pytest.raises(pkg.AcaError) as ei:
        g.run_until(float(t.max()) / 2 ** 32 + 3.0)
    assert ei.value.code == -6
    # a state whose counters cannot fit is refused up front
    n[:] = 2 ** 31
    with pytest.raises(pkg.AcaError) as ei:
        g.set_state(s, t, n)
    assert ei.value.code == -6


def test_set_spins_user_initial_state(aca, oracle_mod):
    import workloads
    sp = workloads.host_spins((64, 64), seed=5)
    g = aca.Sim((64, 64), beta=0.44, seed=3, whole_lattice=-1)
    g.set_spins(sp)
    assert np.array_equal(g.spins().ravel(), sp)


def test_config2_scaled(aca, oracle_mod):
    """Config 2's physics (Metropolis beta 0.40, 64x64 tiles) on 512x512 to T = 8."""
    g, o = run_pair(aca, oracle_mod, (512, 512), [8.0], beta=0.40, rule=1, seed=1, tile=(64, 64))
    assert_same(g, o)


@pytest.mark.parametrize("dims", [(256, 192), (32, 24, 16)])
def test_nccl_transport_ring_of_one(aca, oracle_mod, dims):
    """The multi-process path on one GPU: a 1-rank NCCL communicator built from
    aca_nccl_unique_id, halo rows/planes exchanged with grouped ncclSend/ncclRecv to the ring
    neighbours (here the rank itself), termination all-reduced. Bit-exact vs the oracle."""
    import torch  # noqa: F401  (loads libnccl into the process)
    try:
        uid = aca.aca_nccl_unique_id()
    except aca.AcaError as e:
        pytest.skip("NCCL not loadable: %s" % e)
    beta = 0.2216544 if len(dims) == 3 else 0.4406868
    tile = (16, 16, 16) if len(dims) == 3 else (64, 64)
    g, o = run_pair(aca, oracle_mod, dims, [2.0, 4.0], beta=beta, seed=53, nccl_id=uid, tile=tile)
    assert_same(g, o)


def test_config4_scaled(aca, oracle_mod):
    """Config 4's physics (3-D heat-bath at beta 0.2216544) on 64^3 to T = 3, 2 shards."""
    g, o = run_pair(aca, oracle_mod, (64, 64, 64), [3.0], beta=0.2216544, seed=1, shards=2)
    assert_same(g, o)


@pytest.mark.parametrize("dims", [(96, 80), (20, 16, 12)])
def test_class_histogram(aca, oracle_mod, dims):
    """BKL classes |Gamma_k| of the final configuration, recomputed with
    numpy from the oracle's spins, and the n-fold-way rate sum_k |Gamma_k| p_k."""
    g, o = run_pair(aca, oracle_mod, dims, [4.0], beta=1.0, h=0.1, rule=1, init_q=0.05, seed=47, whole_lattice=-1)
    s = o.spins().astype(np.int64)
    nd = len(dims)
    up = (s > 0).astype(np.int64)
    ones = sum(np.roll(up, sh, axis=ax) for ax in range(nd) for sh in (1, -1))
    z = 2 * nd
    idx = ones + (z + 1) * up
    want = np.bincount(idx.ravel(), minlength=2 * (z + 1))
    st = g.stats()
    assert st["class_hist"][:2 * (z + 1)] == [int(v) for v in want]
    thr = oracle_mod.flip_table(nd, 1.0, 1.0, 0.1, 1)
    rate = sum(int(c) * t / 2 ** 32 for c, t in zip(want, thr))
    assert abs(st["nfold_rate"] - rate) < 1e-6 * max(1.0, rate)


@pytest.mark.parametrize("case", ["whole", "tiny", "tiled", "t32", "t64x32", "shards", "ties", "law2",
                                  "block", "frames", "jacobi", "odd"])
def test_game_of_life(aca, oracle_mod, case):
    """Rule 2 (asynchronous Game of Life, P10): Moore neighbourhood, Conway's
    rule, explicit (t, c) tie-break (no rank bits): bit-identical trajectories on the
    whole-lattice kernel, tiled with ragged tiles (corner halo cells), virtual shards, forced
    ties, another law, a user-set still life, and frames."""
    kw = dict(dims=(200, 150), Ts=[3.0, 6.0], seed=61, rule=2, init_q=0.6, whole_lattice=-1)
    if case == "whole":
        kw.update(dims=(24, 20), whole_lattice=1)
    elif case == "tiny":
        kw.update(dims=(3, 5), whole_lattice=0)
    elif case == "t32":
        kw.update(tile=(32, 32))
    elif case == "t64x32":
        kw.update(tile=(64, 32))
    elif case == "jacobi":
        kw.update(checkerboard=-1)
    elif case == "odd":
        kw.update(dims=(320, 192))
    elif case == "shards":
        kw.update(dims=(128, 96), shards=4)
    elif case == "ties":
        kw.update(tie_bits=30)
    elif case == "law2":
        kw.update(law=2)
    if case == "block":
        dims = (96, 64)
        s = -np.ones((64, 96), np.int8)
        s[10:12, 20:22] = 1
        g = aca.Sim(dims, rule=2, seed=5, whole_lattice=-1)
        g.set_spins(s)
        g.run_until(10.0)
        assert np.array_equal(g.spins(), s) and g.stats()["flips"] == 0
        return
    if case == "frames":
        dims = (130, 70)
        g = aca.Sim(dims, rule=2, seed=7, init_q=0.6, whole_lattice=-1)
        o = oracle_mod.OracleSim(dims, rule=2, seed=7, init_q=0.6)
        got = g.frames(0.5, 1, 6, B=3)
        dq = int(np.floor(0.5 * 4294967296.0 + 0.5))
        for k in range(6):
            o.run_until_q32((1 + k) * dq + 1)
            assert np.array_equal(got[k], o.spins())
        return
    dims, Ts = kw.pop("dims"), kw.pop("Ts")
    g, o = run_pair(aca, oracle_mod, dims, Ts, **kw)
    assert_same(g, o)


@pytest.mark.parametrize("env,tile,dims", [(("ACA_TILE_NT", "256"), (64, 64), (320, 200)),
                                           (("ACA_TILE_NT", "512"), (64, 64), (320, 200))])
def test_ablation_switches_stay_exact(aca, oracle_mod, env, tile, dims, monkeypatch):
    """The group size of a tile shape (ACA_TILE_NT) changes the schedule, never the result."""
    monkeypatch.setenv(*env)
    g, o = run_pair(aca, oracle_mod, dims, [3.0, 6.0], beta=0.4406868, seed=71, tile=tile)
    assert_same(g, o)
