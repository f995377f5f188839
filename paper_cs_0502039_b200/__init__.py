"""Python binding of libaca.so (include/aca.h) — argument marshalling only.

Every step of the simulation runs in the CUDA kernels behind the C ABI; this module only
converts arguments (ctypes) and raises on non-zero return codes. There is no CPU fallback:
if libaca.so is missing or no CUDA device is present the calls fail loudly.

Names follow the C ABI: aca_create, aca_run_until, aca_get_spins/times/counters/stats, ...
`Sim` is a small convenience wrapper over the same calls.
"""
import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_PKG, "libaca.so")

ACA_HEATBATH, ACA_METROPOLIS, ACA_LIFE = 0, 1, 2
ERRORS = {0: "ACA_OK", -1: "ACA_EINVAL", -2: "ACA_ENOMEM", -3: "ACA_ECUDA", -4: "ACA_ENCCL",
          -5: "ACA_ESTATE", -6: "ACA_ERANGE", -7: "ACA_ENODEV"}

# symbols declared in include/aca.h (checked by tests/test_abi.py)
EXPORTS = ["aca_default_options", "aca_create", "aca_run_until", "aca_run_until_q32", "aca_get_spins",
           "aca_get_times", "aca_get_counters", "aca_get_cells", "aca_get_stats", "aca_get_flip_table", "aca_set_state",
           "aca_set_spins", "aca_reset", "aca_nccl_unique_id", "aca_destroy", "aca_last_error", "aca_num_cells", "aca_selftest_philox",
           "aca_selftest_nlog", "aca_selftest_law", "aca_efficiency_run", "aca_run_frames", "aca_agg_run", "aca_bkl_run", "aca_efficiency_run_q", "aca_ipc_export", "aca_ipc_import",
           "aca_stage_spins", "aca_set_spins_staged", "aca_get_spins_async", "aca_sync", "aca_perfbl_run",
           "aca_get_tile_grid", "aca_get_tile_classes", "aca_qnbr_run"]
ACA_IPC_BLOB_BYTES = 192
DEFAULT_ROUNDS = 5   # in-tile rounds per tile visit when aca_options.rounds_per_launch = 0 (aca.cu)
POISSON, UNIFORM, ROOT8, GAUSS = 0, 1, 2, 3   # asynchrony laws (aca_options.law)


class AcaError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("%s: %s" % (ERRORS.get(code, code), msg))
        self.code = code


class aca_options(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_uint32), ("init_q", ctypes.c_double),
                ("tile", ctypes.c_int32 * 3), ("rounds_per_launch", ctypes.c_int32),
                ("launches_per_check", ctypes.c_int32), ("tie_bits", ctypes.c_int32),
                ("sync_rounds", ctypes.c_int32), ("device", ctypes.c_int32), ("shards", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("nccl_id", ctypes.c_void_p),
                ("stream", ctypes.c_void_p), ("event_hash", ctypes.c_int32),
                ("whole_lattice", ctypes.c_int32), ("variant", ctypes.c_int32),
                ("early_reject", ctypes.c_int32), ("checkerboard", ctypes.c_int32),
                ("law", ctypes.c_int32), ("halo_mode", ctypes.c_int32), ("max_ctas", ctypes.c_int32),
                ("lag", ctypes.c_double), ("class_book", ctypes.c_int32), ("class_wmax", ctypes.c_double)]


class aca_qnbr_stats(ctypes.Structure):
    _fields_ = [("arrivals", ctypes.c_uint64), ("flips", ctypes.c_uint64), ("event_hash", ctypes.c_uint64),
                ("bond_sum", ctypes.c_int64), ("magnetisation", ctypes.c_int64), ("launches", ctypes.c_uint64),
                ("sweeps", ctypes.c_uint64), ("gpu_seconds", ctypes.c_double)]


class aca_stats(ctypes.Structure):
    _fields_ = [("arrivals", ctypes.c_uint64), ("flips", ctypes.c_uint64), ("event_hash", ctypes.c_uint64),
                ("bond_sum", ctypes.c_int64), ("magnetisation", ctypes.c_int64), ("t_min", ctypes.c_uint64),
                ("t_max", ctypes.c_uint64), ("launches", ctypes.c_uint64), ("inner_rounds", ctypes.c_uint64),
                ("cells_tested", ctypes.c_uint64), ("cells_fired", ctypes.c_uint64),
                ("gpu_seconds", ctypes.c_double), ("kernel_seconds", ctypes.c_double),
                ("kernel_launches", ctypes.c_uint64), ("time_bits", ctypes.c_int32),
                ("counter_bits", ctypes.c_int32), ("rank_bits", ctypes.c_int32),
                ("class_hist", ctypes.c_uint64 * 14), ("nfold_rate", ctypes.c_double),
                ("tile_visits_early", ctypes.c_uint64), ("tile_visits_plain", ctypes.c_uint64)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["class_hist"] = [int(v) for v in self.class_hist]
        return d


_lib = None


if os.environ.get("ACA_LIB"):   # an alternative build of the same sources (e.g. libaca_dbg.so)
    _SO = os.path.join(os.path.dirname(os.path.abspath(__file__)), os.environ["ACA_LIB"])


def library_path():
    return _SO


def lib():
    """Load libaca.so (building it first if the sources are newer and nvcc is present)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_SO):
        from . import _build
        _build.build()
    L = ctypes.CDLL(_SO)
    vp, i64p = ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)
    L.aca_default_options.argtypes = [ctypes.POINTER(aca_options)]
    L.aca_create.argtypes = [ctypes.POINTER(vp), ctypes.c_int, i64p, ctypes.c_int, ctypes.c_double,
                             ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_uint64,
                             ctypes.POINTER(aca_options)]
    L.aca_run_until.argtypes = [vp, ctypes.c_double]
    L.aca_run_until_q32.argtypes = [vp, ctypes.c_uint64]
    for n in ("aca_get_spins", "aca_get_times", "aca_get_counters", "aca_set_spins"):
        getattr(L, n).argtypes = [vp, vp, ctypes.c_size_t]
    L.aca_get_stats.argtypes = [vp, ctypes.POINTER(aca_stats)]
    L.aca_get_cells.argtypes = [vp, vp, ctypes.c_size_t, vp, vp, vp]
    L.aca_get_flip_table.argtypes = [vp, vp, ctypes.c_size_t]
    L.aca_get_tile_grid.argtypes = [vp, vp]
    L.aca_get_tile_classes.argtypes = [vp, vp, ctypes.c_size_t, ctypes.c_int]
    L.aca_set_state.argtypes = [vp, vp, vp, vp, ctypes.c_size_t]
    L.aca_reset.argtypes = [vp, ctypes.c_uint64]
    L.aca_nccl_unique_id.argtypes = [vp]
    L.aca_destroy.argtypes = [vp]
    L.aca_destroy.restype = None
    L.aca_last_error.restype = ctypes.c_char_p
    L.aca_num_cells.argtypes = [vp]
    L.aca_num_cells.restype = ctypes.c_int64
    L.aca_selftest_philox.argtypes = [ctypes.c_uint64, vp, vp, vp, vp]
    L.aca_selftest_nlog.argtypes = [ctypes.c_uint64, vp, vp, vp, ctypes.c_uint64, ctypes.c_int]
    L.aca_agg_run.argtypes = [vp, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                              ctypes.c_int, ctypes.c_uint64, ctypes.c_double, ctypes.c_double, ctypes.c_int, vp, vp, vp,
                              ctypes.POINTER(aca_agg_stats), ctypes.c_int]
    L.aca_bkl_run.argtypes = L.aca_agg_run.argtypes
    L.aca_qnbr_run.argtypes = [ctypes.c_int, vp, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                               ctypes.c_double, ctypes.c_int, ctypes.c_uint64, ctypes.c_double, ctypes.c_int,
                               ctypes.c_int, ctypes.c_double, ctypes.c_int, vp, vp, vp,
                               ctypes.POINTER(aca_qnbr_stats), ctypes.c_int]
    L.aca_ipc_export.argtypes = [vp, vp, ctypes.c_size_t]
    L.aca_stage_spins.argtypes = [vp, vp, ctypes.c_size_t, ctypes.c_int]
    L.aca_set_spins_staged.argtypes = [vp, ctypes.c_int]
    L.aca_get_spins_async.argtypes = [vp, vp, ctypes.c_size_t]
    L.aca_sync.argtypes = [vp]
    L.aca_ipc_import.argtypes = [vp, vp, ctypes.c_size_t]
    L.aca_efficiency_run_q.argtypes = [ctypes.c_int, vp, ctypes.c_int, ctypes.c_double, ctypes.c_uint64,
                                       ctypes.c_int64, ctypes.c_int, vp, vp, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
    L.aca_run_frames.argtypes = [vp, ctypes.c_double, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, vp]
    L.aca_efficiency_run.argtypes = [ctypes.c_int, vp, ctypes.c_int, ctypes.c_double, ctypes.c_uint64,
                                     ctypes.c_int64, vp, vp, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
    L.aca_perfbl_run.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_uint64,
                                 ctypes.c_int64, vp, vp, vp, ctypes.c_int]
    L.aca_selftest_law.argtypes = [ctypes.c_uint64, vp, ctypes.c_int, ctypes.c_uint64, ctypes.c_int, vp, vp]
    _lib = L
    return L


def _check(rc):
    if rc != 0:
        raise AcaError(rc, lib().aca_last_error().decode())
    return rc


def aca_default_options(**kw):
    o = aca_options()
    _check(lib().aca_default_options(ctypes.byref(o)))
    for k, v in kw.items():
        if k == "tile":
            for i, t in enumerate(v):
                o.tile[i] = int(t)
        elif k == "nccl_id" and isinstance(v, (bytes, bytearray)):
            o._nccl_buf = (ctypes.c_uint8 * 128).from_buffer_copy(bytes(v))   # kept alive with o
            o.nccl_id = ctypes.cast(o._nccl_buf, ctypes.c_void_p)
        else:
            setattr(o, k, v)
    return o


def aca_create(dims, lam=1.0, beta=0.0, J=1.0, h=0.0, rule=ACA_HEATBATH, seed=1, periodic=1, options=None):
    dims = [int(d) for d in dims]
    arr = (ctypes.c_int64 * len(dims))(*dims)
    p = ctypes.c_void_p()
    opt = options if options is not None else aca_default_options()
    _check(lib().aca_create(ctypes.byref(p), len(dims), arr, periodic, lam, beta, J, h, rule, seed,
                            ctypes.byref(opt)))
    return p


def aca_run_until(p, T):
    return _check(lib().aca_run_until(p, float(T)))


def aca_run_until_q32(p, Tq):
    return _check(lib().aca_run_until_q32(p, int(Tq)))


def aca_num_cells(p):
    return int(lib().aca_num_cells(p))


def _ptr(a):
    if hasattr(a, "data_ptr"):          # torch tensor (e.g. pinned host buffer)
        return ctypes.c_void_p(a.data_ptr())
    return ctypes.c_void_p(a.ctypes.data)


def aca_get_spins(p, out=None):
    n = aca_num_cells(p)
    out = np.empty(n, np.int8) if out is None else out
    _check(lib().aca_get_spins(p, _ptr(out), n))
    return out


def aca_get_times(p, out=None):
    n = aca_num_cells(p)
    out = np.empty(n, np.uint64) if out is None else out
    _check(lib().aca_get_times(p, _ptr(out), n))
    return out


def aca_get_counters(p, out=None):
    n = aca_num_cells(p)
    out = np.empty(n, np.uint32) if out is None else out
    _check(lib().aca_get_counters(p, _ptr(out), n))
    return out


def aca_get_cells(p, idx):
    idx = np.ascontiguousarray(idx, np.int64)
    m = idx.size
    s = np.empty(m, np.int8)
    t = np.empty(m, np.uint64)
    n = np.empty(m, np.uint32)
    _check(lib().aca_get_cells(p, _ptr(idx), m, _ptr(s), _ptr(t), _ptr(n)))
    return s, t, n


def aca_get_stats(p):
    s = aca_stats()
    _check(lib().aca_get_stats(p, ctypes.byref(s)))
    return s.as_dict()


def aca_get_flip_table(p, ndim):
    n = 2 * (2 * ndim + 1)
    a = (ctypes.c_uint64 * n)()
    _check(lib().aca_get_flip_table(p, a, n))
    return [int(v) for v in a]


def aca_get_tile_grid(p):
    """(tiles_x, tiles_y, tiles_z, shards, tile_x, tile_y, tile_z)"""
    a = (ctypes.c_int64 * 7)()
    _check(lib().aca_get_tile_grid(p, a))
    return tuple(int(v) for v in a)


def aca_get_tile_classes(p, refresh=0):
    """a10 per-tile BKL class histograms: uint32 array [shards, tiles_z, tiles_y, tiles_x, 16]."""
    tx, ty, tz, G = aca_get_tile_grid(p)[:4]
    out = np.empty((G, tz, ty, tx, 16), np.uint32)
    _check(lib().aca_get_tile_classes(p, _ptr(out), out.size, int(refresh)))
    return out


def aca_set_state(p, spins, times, counters):
    spins = np.ascontiguousarray(spins, np.int8).ravel()
    times = np.ascontiguousarray(times, np.uint64).ravel()
    counters = np.ascontiguousarray(counters, np.uint32).ravel()
    _check(lib().aca_set_state(p, _ptr(spins), _ptr(times), _ptr(counters), spins.size))


def aca_set_spins(p, spins):
    if not hasattr(spins, "data_ptr"):
        spins = np.ascontiguousarray(spins, np.int8).ravel()
        n = spins.size
    else:
        n = spins.numel()
    _check(lib().aca_set_spins(p, _ptr(spins), n))


def _host_spins(spins):
    if not hasattr(spins, "data_ptr"):
        spins = np.ascontiguousarray(spins, np.int8).ravel()
        return spins, spins.size
    return spins, spins.numel()


def aca_stage_spins(p, spins, slot):
    """Enqueue the host-to-device copy of the spins into staging slot 0/1 (returns at once; keep
    `spins` alive, ideally pinned, until aca_sync)."""
    spins, n = _host_spins(spins)
    _check(lib().aca_stage_spins(p, _ptr(spins), n, int(slot)))
    return spins


def aca_set_spins_staged(p, slot):
    _check(lib().aca_set_spins_staged(p, int(slot)))


def aca_get_spins_async(p, out):
    """Enqueue unpacking + device-to-host copy of the spins into `out` (valid after aca_sync)."""
    n = out.numel() if hasattr(out, "data_ptr") else out.size
    _check(lib().aca_get_spins_async(p, _ptr(out), n))


def aca_sync(p):
    _check(lib().aca_sync(p))


def aca_reset(p, seed):
    return _check(lib().aca_reset(p, int(seed)))


def aca_nccl_unique_id():
    buf = (ctypes.c_uint8 * 128)()
    _check(lib().aca_nccl_unique_id(buf))
    return bytes(buf)


def aca_destroy(p):
    if p:
        lib().aca_destroy(p)


def aca_selftest_philox(ctr, key):
    ctr = np.ascontiguousarray(ctr, np.uint32)
    key = np.ascontiguousarray(key, np.uint32)
    n = ctr.shape[0]
    out = np.empty((n, 4), np.uint32)
    ref = np.empty((n, 4), np.uint32)
    _check(lib().aca_selftest_philox(n, _ptr(ctr), _ptr(key), _ptr(out), _ptr(ref)))
    return out, ref


def aca_selftest_nlog(X, lam=1.0, tie_bits=0):
    X = np.ascontiguousarray(X, np.uint64)
    q = np.empty_like(X)
    d = np.empty_like(X)
    inv = int(np.floor(4294967296.0 / lam + 0.5))
    _check(lib().aca_selftest_nlog(X.size, _ptr(X), _ptr(q), _ptr(d), inv, tie_bits))
    return q, d


def aca_selftest_law(X, law, lam=1.0, tie_bits=0):
    X = np.ascontiguousarray(X, np.uint64)
    u = np.empty_like(X)
    d = np.empty_like(X)
    inv = int(np.floor(4294967296.0 / lam + 0.5))
    _check(lib().aca_selftest_law(X.size, _ptr(X), int(law), inv, tie_bits, _ptr(u), _ptr(d)))
    return u, d


class aca_agg_stats(ctypes.Structure):
    _fields_ = [("arrivals", ctypes.c_uint64), ("flips", ctypes.c_uint64), ("event_hash", ctypes.c_uint64),
                ("bond_sum", ctypes.c_int64), ("magnetisation", ctypes.c_int64), ("launches", ctypes.c_uint64),
                ("gpu_seconds", ctypes.c_double)]


def aca_ipc_export(p):
    """This rank's IPC blob (multi-process push mode)."""
    buf = (ctypes.c_uint8 * ACA_IPC_BLOB_BYTES)()
    _check(lib().aca_ipc_export(p, ctypes.cast(buf, ctypes.c_void_p), ACA_IPC_BLOB_BYTES))
    return bytes(buf)


def aca_ipc_import(p, blobs):
    """All ranks' blobs, in rank order (bytes of world x ACA_IPC_BLOB_BYTES)."""
    b = (ctypes.c_uint8 * len(blobs)).from_buffer_copy(blobs)
    _check(lib().aca_ipc_import(p, ctypes.cast(b, ctypes.c_void_p), len(blobs)))


def aca_agg_run(dims, m, T, lam=1.0, beta=0.0, J=1.0, h=0.0, rule=ACA_HEATBATH, seed=1, init_q=0.5, budget=64,
                want_state=True, device=-1, bkl=False):
    """Aggregated Poisson stream (fig:amcpoi) on the GPU, or with bkl=True the modified BKL of
    PAPER.md:1126-1191: (spins[ny, nx], T[ntiles], n[ntiles], stats) — the state arrays are
    None when want_state is False."""
    nx, ny = int(dims[0]), int(dims[1])
    nt = (nx // m) * (ny // m) if nx % m == 0 and ny % m == 0 else 1
    d = (ctypes.c_int64 * 2)(nx, ny)
    sp = np.zeros(nx * ny, np.int8) if want_state else None
    Tt = np.zeros(nt, np.uint64) if want_state else None
    nn = np.zeros(nt, np.uint32) if want_state else None
    st = aca_agg_stats()
    fn = lib().aca_bkl_run if bkl else lib().aca_agg_run
    _check(fn(ctypes.cast(d, ctypes.c_void_p), int(m), float(lam), float(beta), float(J), float(h),
                             int(rule), int(seed), float(init_q), float(T), int(budget),
                             _ptr(sp) if want_state else None, _ptr(Tt) if want_state else None,
                             _ptr(nn) if want_state else None, ctypes.byref(st), int(device)))
    stats = {k: getattr(st, k) for k, _ in st._fields_}
    return (sp.reshape(ny, nx) if want_state else None), Tt, nn, stats


def aca_qnbr_run(dims, q, T, lam=1.0, beta=0.0, J=1.0, h=0.0, rule=ACA_HEATBATH, seed=1, init_q=0.5, tie_bits=0,
                 law=POISSON, rounds=0, want_state=True, device=-1):
    """The Ising model on the q-th degree neighbourhood (P12) on the GPU: (spins, times, counters,
    stats), the arrays shaped dims[::-1] (None when want_state is False)."""
    dims = tuple(int(v) for v in dims)
    N = int(np.prod(dims))
    d = (ctypes.c_int64 * len(dims))(*dims)
    sp = np.zeros(N, np.int8) if want_state else None
    tt = np.zeros(N, np.uint64) if want_state else None
    nn = np.zeros(N, np.uint32) if want_state else None
    st = aca_qnbr_stats()
    _check(lib().aca_qnbr_run(len(dims), ctypes.cast(d, ctypes.c_void_p), int(q), float(lam), float(beta), float(J),
                              float(h), int(rule), int(seed), float(init_q), int(tie_bits), int(law), float(T),
                              int(rounds), _ptr(sp) if want_state else None, _ptr(tt) if want_state else None,
                              _ptr(nn) if want_state else None, ctypes.byref(st), int(device)))
    stats = {k: getattr(st, k) for k, _ in st._fields_}
    shp = dims[::-1]
    if not want_state:
        return None, None, None, stats
    return sp.reshape(shp), tt.reshape(shp), nn.reshape(shp), stats


def aca_run_frames(p, dt, K0, count, B=4):
    """Frames (fig:genout): int8[count, N] of the states at times K dt, K = K0..K0+count-1."""
    n = int(lib().aca_num_cells(p))
    fb = (n + 7) // 8
    bits = np.zeros(count * fb, np.uint8)
    _check(lib().aca_run_frames(p, float(dt), int(K0), int(count), int(B), _ptr(bits)))
    pm = np.unpackbits(bits.reshape(count, fb), axis=1, bitorder="little")[:, :n]
    return np.where(pm > 0, 1, -1).astype(np.int8)


def aca_perfbl_run(px, py, m, rounds, lag=0.0, seed=1, device=-1):
    """fig:perfbl model on the GPU (include/aca.h aca_perfbl_run): (ups per round, h, n)."""
    n = int(px) * int(py)
    ups = np.zeros(max(rounds, 1), np.uint64)
    hh = np.zeros(n, np.uint64)
    nn = np.zeros(n, np.uint32)
    _check(lib().aca_perfbl_run(px, py, m, float(lag), seed, rounds, ups.ctypes.data, hh.ctypes.data, nn.ctypes.data,
                                device))
    return ups[:rounds], hh, nn


def aca_efficiency_run(dims, rounds, law=POISSON, lam=1.0, seed=1, want_times=False, device=-1, q=1):
    """Time-only efficiency model on the GPU: N0 per synchronous
    iteration (uint64[rounds]), the final times if asked, and the device seconds."""
    d = (ctypes.c_int64 * len(dims))(*[int(v) for v in dims])
    fired = np.zeros(rounds, np.uint64)
    n = int(np.prod(dims))
    t = np.zeros(n, np.uint64) if want_times else None
    sec = ctypes.c_double(0.0)
    _check(lib().aca_efficiency_run_q(len(dims), ctypes.cast(d, ctypes.c_void_p), int(law), float(lam), int(seed),
                                      int(rounds), int(q), _ptr(fired), _ptr(t) if want_times else None, int(device),
                                      ctypes.byref(sec)))
    return (fired, t, sec.value) if want_times else (fired, sec.value)


class Sim:
    """Convenience wrapper: one aca_sim handle."""

    def __init__(self, dims, lam=1.0, beta=0.0, J=1.0, h=0.0, rule=ACA_HEATBATH, seed=1, **opts):
        self.dims = tuple(int(d) for d in dims)
        self.ndim = len(self.dims)
        self.options = aca_default_options(**opts)
        self._p = aca_create(self.dims, lam, beta, J, h, rule, seed, options=self.options)

    @property
    def handle(self):
        return self._p

    def close(self):
        if self._p:
            aca_destroy(self._p)
            self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run_until(self, T):
        aca_run_until(self._p, T)

    def reset(self, seed):
        aca_reset(self._p, seed)

    def run_until_q32(self, Tq):
        aca_run_until_q32(self._p, Tq)

    def _shape(self, a):
        n = aca_num_cells(self._p)
        full = int(np.prod(self.dims))
        return a.reshape(self.dims[::-1]) if n == full else a

    def spins(self):
        return self._shape(aca_get_spins(self._p))

    def times(self):
        return self._shape(aca_get_times(self._p))

    def counters(self):
        return self._shape(aca_get_counters(self._p))

    def stats(self):
        return aca_get_stats(self._p)

    def cells(self, idx):
        return aca_get_cells(self._p, idx)

    def flip_table(self):
        return aca_get_flip_table(self._p, self.ndim)

    def tile_classes(self, refresh=0):
        return aca_get_tile_classes(self._p, refresh)

    def set_state(self, spins, times, counters):
        aca_set_state(self._p, spins, times, counters)

    def frames(self, dt, K0, count, B=4):
        f = aca_run_frames(self._p, dt, K0, count, B)
        n, full = aca_num_cells(self._p), int(np.prod(self.dims))
        return f.reshape((count,) + self.dims[::-1]) if n == full else f

    def set_spins(self, spins):
        aca_set_spins(self._p, spins)
