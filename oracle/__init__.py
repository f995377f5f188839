"""Serial CPU oracle (ctypes wrapper over oracle/liboracle.so).

ORACLE / TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this package. It imports nothing from
the product package ``paper_cs_0502039_b200`` and the product never imports it.

The oracle is the plain definition of the trajectory: all arrivals in increasing (t, c)
order from a global priority queue (PAPER.md:196-211 serial procedure with per-cell
streams, Eq. newt1i; uniqueness PAPER.md:596-613). Primitives:
docs/PRIMITIVES.md.
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = [os.path.join(_HERE, "aca_oracle.c")]
_HDR = [os.path.join(_HERE, "aca_oracle.h"), os.path.join(_HERE, "nlog_tables.h"), os.path.join(_HERE, "gauss_tables.h")]

HEATBATH, METROPOLIS = 0, 1


def build(force=False):
    """Compile liboracle.so with plain gcc (no fast-math: P4 needs glibc exp bit-for-bit)."""
    newest = max(os.path.getmtime(p) for p in _SRC + _HDR)
    if not force and os.path.exists(_SO) and os.path.getmtime(_SO) >= newest:
        return _SO
    tmp = _SO + ".tmp%d" % os.getpid()
    cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fno-fast-math", "-o", tmp] + _SRC + ["-lm"]
    subprocess.check_call(cmd)
    os.replace(tmp, _SO)   # atomic: a process that has the old library mapped keeps it
    return _SO


class Stats(ctypes.Structure):
    _fields_ = [("arrivals", ctypes.c_uint64), ("flips", ctypes.c_uint64),
                ("event_hash", ctypes.c_uint64), ("bond_sum", ctypes.c_int64),
                ("magnetisation", ctypes.c_int64), ("t_min", ctypes.c_uint64),
                ("t_max", ctypes.c_uint64), ("rounds", ctypes.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        L.oracle_philox4x32_10.argtypes = [u32p, u32p, u32p]
        L.oracle_nlog_q32.argtypes = [ctypes.c_uint64]
        L.oracle_nlog_q32.restype = ctypes.c_uint64
        L.oracle_delta.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int]
        L.oracle_delta.restype = ctypes.c_uint64
        L.oracle_delta_law.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_int]
        L.oracle_delta_law.restype = ctypes.c_uint64
        L.oracle_law_q32.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int]
        L.oracle_law_q32.restype = ctypes.c_uint64
        L.oracle_inv_lambda.argtypes = [ctypes.c_double]
        L.oracle_inv_lambda.restype = ctypes.c_uint64
        L.oracle_flip_table.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_int, ctypes.POINTER(ctypes.c_uint64)]
        L.oracle_ev_hash.argtypes = [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int]
        L.oracle_ev_hash.restype = ctypes.c_uint64
        L.oracle_create.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.c_double,
                                    ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                    ctypes.c_uint64, ctypes.c_double, ctypes.c_int]
        L.oracle_create.restype = ctypes.c_void_p
        L.oracle_create_law.argtypes = L.oracle_create.argtypes + [ctypes.c_int]
        L.oracle_create_law.restype = ctypes.c_void_p
        L.oracle_create_q.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.c_int, ctypes.c_double,
                                      ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                      ctypes.c_uint64, ctypes.c_double, ctypes.c_int, ctypes.c_int]
        L.oracle_create_q.restype = ctypes.c_void_p
        L.oracle_q_offsets.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
        L.oracle_q_offsets.restype = ctypes.c_int
        L.oracle_neighbours.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
        L.oracle_neighbours.restype = ctypes.c_int
        L.oracle_flip_table_z.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                          ctypes.c_double, ctypes.c_int, ctypes.POINTER(ctypes.c_uint64)]
        L.oracle_destroy.argtypes = [ctypes.c_void_p]
        L.oracle_run_until_q32.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
        L.oracle_run_until_random_order.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64]
        L.oracle_run_until_calendar.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
        L.oracle_run_until_sync.argtypes = [ctypes.c_void_p, ctypes.c_uint64,
                                            ctypes.POINTER(ctypes.c_uint64), ctypes.c_int64]
        L.oracle_run_until_sync.restype = ctypes.c_int64
        L.oracle_run_until_sync_naive_leq.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
        L.oracle_run_until_sync_naive_leq.restype = ctypes.c_int64
        L.oracle_get_spins.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_set_spins.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_get_times.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_get_counters.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_get_stats.argtypes = [ctypes.c_void_p, ctypes.POINTER(Stats)]
        L.oracle_num_cells.argtypes = [ctypes.c_void_p]
        L.oracle_num_cells.restype = ctypes.c_int64
        L.oracle_replica_hist.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.c_double,
                                          ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_uint64,
                                          ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p]
        L.oracle_time_weighted_hist.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int64),
                                                ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                                ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                                ctypes.c_uint64, ctypes.c_void_p]
        L.oracle_nlog_batch.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_cell_time_counter.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                               ctypes.c_uint64, ctypes.c_int,
                                               ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint32)]
        L.oracle_cell_time_counter_law.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                                   ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                                                   ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint32)]
        L.oracle_window_cell.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.c_double,
                                         ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                         ctypes.c_uint64, ctypes.c_double, ctypes.c_int, ctypes.c_uint64,
                                         ctypes.POINTER(ctypes.c_int64), ctypes.c_int64, ctypes.c_int,
                                         ctypes.POINTER(ctypes.c_int8), ctypes.POINTER(ctypes.c_uint64),
                                         ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_int)]
        L.oracle_window_cell_law.argtypes = L.oracle_window_cell.argtypes + [ctypes.c_int]
        L.oracle_agg_run.argtypes = [ctypes.POINTER(ctypes.c_int64), ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_uint64, ctypes.c_double,
                                     ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.POINTER(Stats)]
        L.oracle_bkl_run.argtypes = L.oracle_agg_run.argtypes
        L.oracle_gauss_z.argtypes = [ctypes.c_uint32]
        L.oracle_gauss_z.restype = ctypes.c_double
        L.oracle_gauss_u.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32]
        L.oracle_gauss_u.restype = ctypes.c_uint64
        L.oracle_cell_period_q32.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.oracle_cell_period_q32.restype = ctypes.c_uint64
        L.oracle_perfbl_run.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                         ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_efficiency_run_q.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.c_int,
                                              ctypes.c_double, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int,
                                              ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_efficiency_run.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.c_int,
                                            ctypes.c_double, ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p,
                                            ctypes.c_void_p]
        _lib = L
    return _lib


def to_q32(T):
    """P6: T_q32 = floor(T * 2^32 + 0.5) in IEEE double."""
    return int(np.floor(np.float64(T) * np.float64(4294967296.0) + np.float64(0.5)))


def philox(ctr, key):
    c = (ctypes.c_uint32 * 4)(*ctr)
    k = (ctypes.c_uint32 * 2)(*key)
    o = (ctypes.c_uint32 * 4)()
    lib().oracle_philox4x32_10(c, k, o)
    return tuple(o)


def nlog_q32(X):
    return lib().oracle_nlog_q32(X)


def nlog_batch(X):
    X = np.ascontiguousarray(X, np.uint64)
    q = np.empty_like(X)
    lib().oracle_nlog_batch(X.size, X.ctypes.data, q.ctypes.data)
    return q


POISSON, UNIFORM, ROOT8, GAUSS, GAUSS_CELL = 0, 1, 2, 3, 4   # P3L asynchrony laws


def cell_time_counter(seed, c, T, lam=1.0, tie_bits=0, law=POISSON):
    """(t, n) of cell c after run_until(T) from its own stream (state independence)."""
    t = ctypes.c_uint64()
    n = ctypes.c_uint32()
    lib().oracle_cell_time_counter_law(seed, c, to_q32(T), lib().oracle_inv_lambda(lam), tie_bits, law,
                                       ctypes.byref(t), ctypes.byref(n))
    return t.value, n.value


def delta(w1, w2, lam=1.0, tie_bits=0, law=POISSON):
    return lib().oracle_delta_law(w1, w2, lib().oracle_inv_lambda(lam), tie_bits, law)


def law_q32(w1, w2, law):
    return lib().oracle_law_q32(w1, w2, law)


def gauss_z(w):
    """The normal quantile of (w + 1/2) 2^-32 as P3L defines it (double)."""
    return lib().oracle_gauss_z(w)


def gauss_u(w, sa, sb, tag):
    return lib().oracle_gauss_u(w, sa, sb, tag)


def cell_period_q32(seed, c):
    """Law 4: the fixed Gaussian period of cell c (Q32)."""
    return lib().oracle_cell_period_q32(seed, c)


def flip_table(ndim, beta, J=1.0, h=0.0, rule=HEATBATH):
    n = 2 * (2 * ndim + 1)
    out = (ctypes.c_uint64 * n)()
    lib().oracle_flip_table(ndim, beta, J, h, rule, out)
    return [int(v) for v in out]


def flip_table_z(zc, beta, J=1.0, h=0.0, rule=HEATBATH):
    """P4 table for zc neighbours (2 (zc + 1) entries); zc = |neighbors^q| - 1 for P12."""
    out = (ctypes.c_uint64 * (2 * (zc + 1)))()
    lib().oracle_flip_table_z(zc, beta, J, h, rule, out)
    return [int(v) for v in out]


def q_offsets(ndim, q):
    """Eq. neiq as the oracle applies it: the offsets of neighbors^q(c) minus c."""
    out = (ctypes.c_int * (3 * 256))()
    n = lib().oracle_q_offsets(ndim, q, out, 256)
    if n < 0:
        raise ValueError("too many offsets")
    return [tuple(out[3 * i:3 * i + ndim]) for i in range(n)]


def ev_hash(w3, t, l, new_spin):
    """P7 event hash term of one arrival."""
    return lib().oracle_ev_hash(w3, t, l, new_spin)


def _dims(dims):
    return (ctypes.c_int64 * len(dims))(*dims)


class OracleSim:
    """One serial simulation. Methods mirror the C-ABI names of the product path."""

    def __init__(self, dims, lam=1.0, beta=0.0, J=1.0, h=0.0, rule=HEATBATH, seed=1,
                 init_q=0.5, tie_bits=0, law=POISSON, q=1):
        self.dims = tuple(int(d) for d in dims)
        self.ndim = len(self.dims)
        self.q = int(q)
        self._p = lib().oracle_create_q(self.ndim, _dims(self.dims), self.q, lam, beta, J, h, rule,
                                        seed, init_q, tie_bits, law)
        if not self._p:
            raise ValueError("oracle_create rejected the arguments")
        self.N = int(np.prod(self.dims))

    def close(self):
        if self._p:
            lib().oracle_destroy(self._p)
            self._p = None

    def __del__(self):
        self.close()

    def run_until(self, T, order="pq", choice_seed=0):
        return self.run_until_q32(to_q32(T), order, choice_seed)

    def run_until_q32(self, Tq, order="pq", choice_seed=0, fired_per_round=None):
        if order == "pq":
            rc = lib().oracle_run_until_q32(self._p, Tq)
        elif order == "calendar":   # (D): the same queue as "pq", bucketed
            rc = lib().oracle_run_until_calendar(self._p, Tq)
            if rc == -2:
                raise MemoryError("calendar queue allocation")
        elif order == "random":
            rc = lib().oracle_run_until_random_order(self._p, Tq, choice_seed)
        elif order == "sync":
            buf = None
            if fired_per_round is not None:
                buf = fired_per_round.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))
            rc = lib().oracle_run_until_sync(self._p, Tq, buf,
                                             0 if fired_per_round is None else len(fired_per_round))
            return rc
        elif order == "naive_leq":   # negative control only
            return lib().oracle_run_until_sync_naive_leq(self._p, Tq)
        else:
            raise ValueError(order)
        if rc != 0:
            raise ValueError("T decreased")
        return rc

    def set_spins(self, spins):
        a = np.ascontiguousarray(np.asarray(spins, np.int8).ravel())
        assert a.size == self.N
        lib().oracle_set_spins(self._p, a.ctypes.data)

    def spins(self):
        a = np.empty(self.N, np.int8)
        lib().oracle_get_spins(self._p, a.ctypes.data)
        return a.reshape(self.dims[::-1])

    def times(self):
        a = np.empty(self.N, np.uint64)
        lib().oracle_get_times(self._p, a.ctypes.data)
        return a.reshape(self.dims[::-1])

    def counters(self):
        a = np.empty(self.N, np.uint32)
        lib().oracle_get_counters(self._p, a.ctypes.data)
        return a.reshape(self.dims[::-1])

    def neighbours(self, c):
        """The cells whose spins enter Sigma(c) and whose (t, c) gate c's arrival."""
        out = (ctypes.c_int64 * 128)()
        n = lib().oracle_neighbours(self._p, int(c), out)
        return [int(out[i]) for i in range(n)]

    def stats(self):
        s = Stats()
        lib().oracle_get_stats(self._p, ctypes.byref(s))
        return s.as_dict()


def replica_hist(dims, beta, J=1.0, h=0.0, rule=HEATBATH, seed0=1, n_rep=1000, T=50.0):
    n = int(np.prod(dims))
    hist = np.zeros(1 << n, np.uint64)
    rc = lib().oracle_replica_hist(len(dims), _dims(dims), beta, J, h, rule, seed0, n_rep,
                                   to_q32(T), hist.ctypes.data)
    assert rc == 0
    return hist


def time_weighted_hist(dims, beta, J=1.0, h=0.0, rule=HEATBATH, seed=1, T0=50.0, T1=1000.0):
    n = int(np.prod(dims))
    w = np.zeros(1 << n, np.float64)
    rc = lib().oracle_time_weighted_hist(len(dims), _dims(dims), beta, J, h, rule, seed,
                                         to_q32(T0), to_q32(T1), w.ctypes.data)
    assert rc == 0
    return w


def window_cell(dims, center, T, radius, lam=1.0, beta=0.0, J=1.0, h=0.0, rule=HEATBATH, seed=1, init_q=0.5,
                tie_bits=0, refine=True, law=POISSON):
    """Exact (s, t, n, exact) of the cell at `center` (x, y[, z]) after run_until(T), from a
    box of the given radius (light-cone oracle; see aca_oracle.c). exact=False: enlarge."""
    so, to, no, ex = ctypes.c_int8(), ctypes.c_uint64(), ctypes.c_uint32(), ctypes.c_int()
    rc = lib().oracle_window_cell_law(len(dims), _dims(dims), lam, beta, J, h, rule, seed, init_q, tie_bits,
                                      to_q32(T), _dims(center), radius, 1 if refine else 0, ctypes.byref(so),
                                      ctypes.byref(to), ctypes.byref(no), ctypes.byref(ex), law)
    assert rc == 0
    return so.value, to.value, no.value, bool(ex.value)


def efficiency_run(dims, rounds, law=POISSON, lam=1.0, seed=1, want_times=False, q=1):
    """Time-only model of PAPER.md:1355-1442 (q-th degree neighbourhood, Eq. neiq): N0 per
    synchronous iteration (and final times)."""
    n = int(np.prod(dims))
    fired = np.zeros(rounds, np.uint64)
    t = np.zeros(n, np.uint64) if want_times else None
    rc = lib().oracle_efficiency_run_q(len(dims), _dims(dims), law, lam, seed, rounds, q, fired.ctypes.data,
                                       t.ctypes.data if want_times else None)
    assert rc == 0
    return (fired, t) if want_times else fired


def perfbl_run(px, py, m, rounds, lag=0.0, seed=1):
    """fig:perfbl model (docs/PRIMITIVES.md P11): PEs that advanced
    in each round, final h (Q32) and n. lag in units of a cell's mean inter-arrival time
    (0 = unbounded)."""
    N = int(px) * int(py)
    ups = np.zeros(rounds, np.uint64)
    hh = np.zeros(N, np.uint64)
    nn = np.zeros(N, np.uint32)
    rc = lib().oracle_perfbl_run(px, py, m, to_q32(lag) if lag else 0, seed, rounds, ups.ctypes.data, hh.ctypes.data,
                                 nn.ctypes.data)
    assert rc == 0
    return ups, hh, nn


def agg_run(dims, m, T, lam=1.0, beta=0.0, J=1.0, h=0.0, rule=HEATBATH, seed=1, init_q=0.5, bkl=False):
    """Aggregated Poisson stream (fig:amcpoi), or with bkl=True the modified BKL of
    PAPER.md:1126-1191: spins[ny, nx], T[ntiles], n[ntiles], stats."""
    nx, ny = int(dims[0]), int(dims[1])
    nt = (nx // m) * (ny // m)
    sp = np.zeros(nx * ny, np.int8)
    Tt = np.zeros(nt, np.uint64)
    nn = np.zeros(nt, np.uint32)
    st = Stats()
    fn = lib().oracle_bkl_run if bkl else lib().oracle_agg_run
    rc = fn(_dims(dims), m, lam, beta, J, h, rule, seed, init_q, to_q32(T), sp.ctypes.data,
            Tt.ctypes.data, nn.ctypes.data, ctypes.byref(st))
    if rc != 0:
        raise ValueError("oracle_agg_run rejected the arguments")
    return sp.reshape(ny, nx), Tt, nn, st.as_dict()
