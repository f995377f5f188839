"""a10 per-tile class bookkeeping (aca_options.class_book, north_star "per-tile
Bortz-Kalos-Lebowitz n-fold-way class bookkeeping (5 neighbour-sum classes x 2 spin states)").

Every tile visit recounts the BKL classes (s, Sigma) of the tile's cells
when it writes them back; the next visit of the tile takes the a10 early-rejection path iff the
tile's mean flip probability per arrival, sum_k |Gamma_k| p_k / cells (the n-fold-way rate,
PAPER.md:1049-1060), is at most class_wmax. Both paths are exact, so:
  * the trajectory stays bit-identical to the serial oracle for every threshold (never, some
    tiles, always), ragged tiles, a capped grid and virtual shards;
  * the per-tile histograms equal a numpy recount of the oracle's final spins: all tiles after
    a refresh, and without one the tiles of the last checkerboard colour (their last visit came
    after every other change);
  * the path counters follow the threshold.
"""
import numpy as np
import pytest

from test_gpu_parity import aca, assert_same, run_pair  # noqa: F401  (fixture + helpers)

pytestmark = pytest.mark.gpu

C5 = dict(beta=1.0, h=0.1, rule=1, init_q=0.05)


def recount(spins, tile):
    """Per-tile class histograms [tz, ty, tx, 16] of a row-major spin array (numpy, from the
    definition: class = (#+1 neighbours) + (z + 1) [s = +1], periodic)."""
    s = np.asarray(spins)
    nd = s.ndim
    up = (s > 0).astype(np.int64)
    ones = sum(np.roll(up, sh, axis=ax) for ax in range(nd) for sh in (1, -1))
    cls = ones + (2 * nd + 1) * up
    if nd == 2:
        cls = cls[None]
        tile = (tile[0], tile[1], 1)
    nz, ny, nx = cls.shape
    tz, ty, tx = -(-nz // tile[2]), -(-ny // tile[1]), -(-nx // tile[0])
    out = np.zeros((tz, ty, tx, 16), np.int64)
    for k in range(tz):
        for j in range(ty):
            for i in range(tx):
                blk = cls[k * tile[2]:(k + 1) * tile[2], j * tile[1]:(j + 1) * tile[1], i * tile[0]:(i + 1) * tile[0]]
                out[k, j, i] = np.bincount(blk.ravel(), minlength=16)
    return out


CASES = {
    "c5_never": dict(dims=(256, 256), Ts=[20.0], class_wmax=-1.0, **C5),
    "c5_some": dict(dims=(256, 256), Ts=[8.0, 20.0], class_wmax=0.002, **C5),
    "c5_always": dict(dims=(256, 256), Ts=[20.0], class_wmax=1.0, **C5),
    "hb_some": dict(dims=(256, 256), Ts=[5.0], beta=0.6, h=0.05, rule=0, class_wmax=0.05),
    "ragged": dict(dims=(200, 136), Ts=[6.0], class_wmax=0.002, **C5),
    "capped": dict(dims=(512, 256), Ts=[6.0], class_wmax=0.002, max_ctas=3, **C5),
    "shards": dict(dims=(256, 256), Ts=[6.0], class_wmax=0.002, shards=2, **C5),
    "ties": dict(dims=(256, 128), Ts=[8.0], class_wmax=0.01, tie_bits=30, **C5),
    "3d": dict(dims=(64, 32, 32), Ts=[4.0], beta=0.5, h=0.1, rule=1, init_q=0.05, class_wmax=0.01),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_class_book_exact(aca, oracle_mod, case):
    kw = dict(CASES[case])
    dims, Ts = kw.pop("dims"), kw.pop("Ts")
    g, o = run_pair(aca, oracle_mod, dims, Ts, seed=61, early_reject=1, class_book=1, **kw)
    assert_same(g, o)
    st = g.stats()
    if kw["class_wmax"] < 0:
        assert st["tile_visits_early"] == 0 and st["tile_visits_plain"] > 0
    elif kw["class_wmax"] >= 1:
        assert st["tile_visits_plain"] == 0 and st["tile_visits_early"] > 0
    else:
        assert st["tile_visits_early"] + st["tile_visits_plain"] > 0
    # the histograms against the oracle's final configuration
    grid = aca.aca_get_tile_grid(g.handle)
    tile = grid[4:7]
    want = recount(o.spins(), tile)
    got = g.tile_classes(refresh=1)
    G = grid[3]
    assert np.array_equal(np.concatenate(list(got), axis=0 if len(dims) == 3 else 1), want), "refreshed histograms"
    # the n-fold rate of the tiles adds up to the whole lattice's
    thr = oracle_mod.flip_table(len(dims), kw.get("beta", 0.4406868), 1.0, kw.get("h", 0.0), kw.get("rule", 0))
    p = np.array([t / 2 ** 32 for t in thr] + [0.0] * (16 - len(thr)))
    assert abs(float((want * p).sum()) - st["nfold_rate"]) < 1e-6 * max(1.0, st["nfold_rate"])
    assert G >= 1


@pytest.mark.parametrize("dims,Ts,extra", [
    ((256, 256), [20.0], {}), ((256, 192), [5.0, 9.0], {}), ((64, 64, 32), [3.0], {}),
    # the 2-D bit-sliced recount: many visits per group (both bitmap parities, the buffer ring),
    # a disordered heat-bath state (every class populated), ragged edge tiles
    ((512, 512), [4.0, 7.0], dict(max_ctas=3, beta=0.35, rule=0, init_q=0.5, class_wmax=0.05)),
    ((520, 264), [6.0], dict(beta=0.5, rule=0, init_q=0.5, class_wmax=-1.0)),
])
def test_kernel_histograms_of_the_last_colour(aca, oracle_mod, dims, Ts, extra):
    """Without a refresh: each tile of the colour launched last was recounted by the tile kernel
    at its final visit, after which nothing changed, so it equals the recount of the oracle's
    final spins; every tile's histogram counts exactly its cells."""
    kw = dict(beta=1.0 if len(dims) == 2 else 0.5, h=0.1, rule=1, init_q=0.05, class_wmax=0.002)
    kw.update(extra)
    g, o = run_pair(aca, oracle_mod, dims, Ts, seed=67, early_reject=1, class_book=1, **kw)
    assert_same(g, o)
    tx, ty, tz, G, *tile = aca.aca_get_tile_grid(g.handle)
    assert G == 1
    got = g.tile_classes(refresh=0)[0]
    want = recount(o.spins(), tile)
    cells = want.sum(axis=3)
    assert np.array_equal(got.sum(axis=3), cells)
    par = (np.arange(tz)[:, None, None] + np.arange(ty)[None, :, None] + np.arange(tx)[None, None, :]) & 1
    last = par == 1
    assert last.any()
    assert np.array_equal(got[last], want[last])


def test_class_book_errors(aca):
    with pytest.raises(aca.AcaError):
        aca.Sim((128, 128), beta=1.0, class_book=1, tile=(32, 32, 1))     # no class instance for this shape
    with pytest.raises(aca.AcaError):
        aca.Sim((128, 128), beta=1.0, class_book=1, sync_rounds=1)
    g = aca.Sim((128, 128), beta=1.0, whole_lattice=-1)
    with pytest.raises(aca.AcaError):
        g.tile_classes()                                                   # bookkeeping off
    g.close()


@pytest.mark.parametrize("opts", [dict(early_reject=1, class_book=1, class_wmax=1.0),
                                  dict(early_reject=1, class_book=0),
                                  dict(early_reject=1, class_book=1, class_wmax=0.002),
                                  dict(early_reject=0, class_book=0)])
def test_high_half_ties_fast_paths(aca, oracle_mod, monkeypatch, opts):
    """The fast arrival (Poisson, lambda = 1, no tie stress) with frequent equal high halves: a
    10-bit counter field leaves the words' high halves a time quantum of 2^-10, so the a10 and
    plain tests meet tied neighbours on a small lattice (their exact passes and the strict rounds'
    conservative treatment), as c5 does at 8192^2."""
    monkeypatch.setenv("ACA_NB_CAP", "10")
    g, o = run_pair(aca, oracle_mod, (256, 256), [10.0, 25.0], seed=71, **C5, **opts)
    assert_same(g, o)
