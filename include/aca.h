/* aca.h — C ABI of the B200-native conservative simulator of Poisson-asynchronous
 * cellular arrays (Lubachevsky, "Efficient Parallel Simulations of Asynchronous Cellular
 * Arrays", arXiv cs/0502039; the reference text is PAPER.md).
 *
 * The calls follow the paper's problem statement: a periodic lattice of cells, each with a
 * state s(c) and a local time t(c); Poisson arrivals of rate lambda
 * (Eq. newt1i); next_state from the neighbourhood just before the arrival
 * (Eq. newst), here continuous-time Glauber / Metropolis Ising
 * (Appendix); simulate until end_time
 * (fig:a1c1pe). All arithmetic on the path is integer (the optional Gaussian laws
 * add correctly rounded IEEE double steps that host and device perform identically) and follows
 * docs/PRIMITIVES.md (P1 Philox4x32-10, P3 NLOG-2, P4 threshold table, P5 init, P6 (t, c)
 * tie-break, P7 event hash), so results are bit-identical to the serial oracle for every
 * tile shape, rounds-per-launch and shard count.
 *
 * Conventions
 *   - Return codes: ACA_OK (0) or a negative ACA_E* code; aca_last_error() then returns a
 *     thread-local message. No function throws across the ABI.
 *   - Host buffers passed to getters/setters are owned by the caller; `count` must equal
 *     the number of cells of the handle (whole lattice; for a multi-process handle the
 *     rank's own rows), else ACA_EINVAL. Layout: row-major, x fastest:
 *     c = y*nx + x (2-D), c = (z*ny + y)*nx + x (3-D).
 *   - All device memory is owned by the library (cudaMalloc at create, freed by destroy).
 *   - Getters synchronise the handle's stream. One handle per host thread at a time.
 *   - There is no CPU fallback: without a CUDA device aca_create returns ACA_ENODEV.
 */
#ifndef ACA_H
#define ACA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct aca_sim aca_sim; /* opaque, library-owned */

/* next_state rules: Glauber heat-bath and Metropolis Ising (P4), and rule 2, the asynchronous
 * Game of Life (P10): Conway's B3/S23 rule on the Moore neighbourhood, a
 * deterministic next_state (2-D only; the Philox draw then only gives the increment). */
enum { ACA_HEATBATH = 0, ACA_METROPOLIS = 1, ACA_LIFE = 2 };

enum {
    ACA_OK = 0,
    ACA_EINVAL = -1, /* invalid argument (message names it) */
    ACA_ENOMEM = -2, /* device or host allocation failed */
    ACA_ECUDA = -3,  /* a CUDA call failed (message has the CUDA error string) */
    ACA_ENCCL = -4,  /* NCCL unavailable or a NCCL call failed */
    ACA_ESTATE = -5, /* call out of order (e.g. T decreased) or invariant violated */
    ACA_ERANGE = -6, /* times would overflow the packed 64-bit word */
    ACA_ENODEV = -7  /* no CUDA device */
};

typedef struct {
    uint32_t struct_size;       /* = sizeof(aca_options); checked */
    double init_q;              /* P5: probability that s0(c) = -1 (default 0.5) */
    int32_t tile[3];            /* CTA tile (x, y, z); 0 = default (64x64, 32x16x8) */
    int32_t rounds_per_launch;  /* R_max in-tile rounds per tile visit (0 = default 5) */
    int32_t launches_per_check; /* K launches between host checks of termination (0 = 16) */
    int32_t tie_bits;           /* P3b tie-stress quantisation (0 = off) */
    int32_t sync_rounds;        /* 1: exact fig:s1c1pe two-phase rounds */
    int32_t device;             /* CUDA device ordinal; -1 = current device */
    int32_t shards;             /* virtual row/plane shards on this device (default 1) */
    int32_t rank, world;        /* multi-process strips: this rank of `world` (default 0, 1) */
    const void* nccl_id;        /* world > 1 with halo_mode 1: 128-byte ncclUniqueId shared by
                                   all ranks (halo rows by NCCL send/recv). world 1: a ring of
                                   one through NCCL (transport test). Unused in push mode. */
    void* stream;               /* cudaStream_t to run on; NULL = library-owned stream */
    int32_t event_hash;         /* 1 (default): accumulate the P7 event hash */
    int32_t whole_lattice;      /* 1: one CTA holds the whole lattice with periodic
                                   addressing and runs to completion in one launch
                                   (small lattices, config 1); 0 = auto, -1 = never */
    int32_t variant;            /* must be 0. Round 1's kernel ablations (uncompacted tiles,
                                   double-buffered TMA, register-resident rounds, work lists,
                                   2-wide halos) were measured slower and retired; DESIGN.md
                                   section 6 keeps their numbers. The group size of the 64x64
                                   tile is chosen by the library (512 threads when a launch has
                                   fewer than two tiles per SM). Environment switches for
                                   ablations only: ACA_TILE_NT, ACA_BULK, ACA_EFF_STREAM,
                                   ACA_NO_RES, ACA_RES_NT, ACA_NO_TMA_BOX, ACA_TMA_PROMO; for tests only:
                                   ACA_NB_CAP=b caps the counter field at b bits (the words'
                                   high halves then tie often: exercises the exact passes). */
    int32_t early_reject;       /* 1: a cell may also commit arrivals that are rejected for
                                   every possible state of the neighbours it still waits for
                                   (exact; pays off at low temperature, config 5). 0 = off */
    int32_t checkerboard;       /* persistent tile kernels: 0 (default) / 1 = each sweep is two
                                   launches, the tiles of one checkerboard colour each (no two
                                   tiles of a launch are adjacent, so every tile reads its
                                   neighbours' state of the same sweep: Gauss-Seidel across
                                   tiles); -1 = one launch over all tiles. Same results. */
    int32_t law;                /* asynchrony law of the increments (docs/PRIMITIVES.md P3L):
                                   0 (default) Poisson, next_t = t - ln(r)/lambda (Eq. newt1i,
                                   PAPER.md:485-488); 1 uniform, next_t - t = r/lambda
                                   (PAPER.md:1389-1393); 2 next_t - t = r^(1/8)/lambda
                                   (PAPER.md:1425-1430); 3 a Gaussian period of mean 1/lambda and
                                   sd 1/(4 lambda) drawn at every arrival (the normal quantile of
                                   r, periods below one unit redrawn); 4 the
                                   strict reading of PAPER.md:404-410: a fixed Gaussian period per
                                   cell. r from the arrival's draw (law 4: the cell's initial draw). */
    int32_t halo_mode;          /* sharded handles: 0 (default) = push, the tile kernel stores its
                                   boundary rows into the neighbour shard's halo as it writes them
                                   back (no exchange step; exact because words only grow and are
                                   never torn); 1 = exchange the halo rows before every launch
                                   (device copies / NCCL send-recv). Same results. world > 1
                                   with 0: the neighbours' halos are mapped by CUDA IPC
                                   (aca_ipc_export / aca_ipc_import below). */
    int32_t max_ctas;           /* > 0: cap the persistent tile kernel's grid (default 0 = one
                                   CTA per SM). Small caps make every CTA cycle many tiles
                                   through its buffer ring (tests of that path on small
                                   lattices). Same results. */
    double lag;                 /* > 0: bounded lag: a launch fires only
                                   arrivals below min(T, t_min + lag/lambda), t_min the minimum
                                   pending time when the launch starts (per shard after the first
                                   launch of a run_until), lag in units of a cell's mean
                                   inter-arrival time 1/lambda. A scheduling
                                   bound only: same results; 0 (default) = unbounded. Not with
                                   multi-process handles. */
    int32_t class_book;         /* 1: per-tile BKL class bookkeeping (a10 as north_star words it;
                                   classes (s, Sigma) in the P4 index): every
                                   tile visit recounts the classes of the tile's cells when it
                                   writes them back, and each visit of a tile takes the a10
                                   early-rejection path (with early_reject = 1) iff the tile's
                                   mean flip probability per arrival at its last visit,
                                   sum_k |Gamma_k| p_k / cells (the n-fold-way rate per cell over
                                   lambda), is at most class_wmax; otherwise
                                   the plain test. Both paths are exact: same results. Needs the
                                   default tile shape and an Ising rule. 0 (default) = off. */
    double class_wmax;          /* see class_book; < 0 = never the a10 path, >= 1 = always */
} aca_options;

typedef struct {
    uint64_t arrivals;      /* sum_c n(c) */
    uint64_t flips;         /* arrivals that changed the spin */
    uint64_t event_hash;    /* P7 */
    int64_t bond_sum;       /* B = sum_c s(c) sum_a s(c + e_a) (periodic) */
    int64_t magnetisation;  /* M = sum_c s(c) */
    uint64_t t_min, t_max;  /* over pending arrival times, Q32 */
    uint64_t launches;      /* tile-kernel launches that did work */
    uint64_t inner_rounds;  /* sum over launches of the max in-tile rounds executed */
    uint64_t cells_tested;  /* eligibility tests of cells with t < T */
    uint64_t cells_fired;   /* = arrivals processed by the kernels */
    double gpu_seconds;     /* CUDA-event time inside aca_run_until calls */
    double kernel_seconds;  /* CUDA-event time of the kernel batches alone */
    uint64_t kernel_launches; /* every tile-kernel launch issued (incl. no-op tail) */
    int32_t time_bits, counter_bits, rank_bits; /* current split of the packed state word */
    uint64_t class_hist[14];  /* BKL classes |Gamma_k| of the current configuration, index
                                 (Sigma+z)/2 + (z+1)(s+1)/2 as the P4 table */
    double nfold_rate;        /* lambda * sum_k |Gamma_k| p_k: the total flip rate of the BKL
                                 n-fold way */
    uint64_t tile_visits_early; /* class_book: tile visits that took the a10 path ... */
    uint64_t tile_visits_plain; /* ... and the plain test (0 without class_book) */
} aca_stats;

/* Fill *opt with defaults (struct_size set). */
int aca_default_options(aca_options* opt);

/* Create a simulation and initialise it on the device (P5: one Philox draw per cell).
 * ndim in {2, 3}; dims[a] >= 2; periodic must be 1;
 * lambda > 0 finite; beta >= 0 finite; rule ACA_HEATBATH, ACA_METROPOLIS or (2-D) ACA_LIFE;
 * opt may be NULL (defaults). On success *out owns device memory until aca_destroy. */
int aca_create(aca_sim** out, int ndim, const int64_t* dims, int periodic, double lambda,
               double beta, double J, double h, int rule, uint64_t seed, const aca_options* opt);

/* Process every arrival with t < T (strict). T_q32 = floor(T*2^32 + 0.5).
 * Successive calls must have non-decreasing T (else ACA_ESTATE) and compose exactly. */
int aca_run_until(aca_sim* s, double T);
int aca_run_until_q32(aca_sim* s, uint64_t T_q32);

/* Copy the current state to caller-owned host memory (count = cells). */
int aca_get_spins(aca_sim* s, int8_t* out, size_t count);
int aca_get_times(aca_sim* s, uint64_t* out, size_t count);   /* pending arrival, Q32 */
int aca_get_counters(aca_sim* s, uint32_t* out, size_t count); /* n(c) */
/* Sampled cells: for i < m, cell idx[i] (row-major, handle-local) -> spins[i], times[i],
 * counters[i]; any output pointer may be NULL. Gathered on the device (no full copy). */
int aca_get_cells(aca_sim* s, const int64_t* idx, size_t m, int8_t* spins, uint64_t* times,
                  uint32_t* counters);
/* Statistics (device reductions; synchronises). */
int aca_get_stats(aca_sim* s, aca_stats* out);
/* P4 table: count = 10 (2-D) or 14 (3-D), index (Sigma+z)/2 + (z+1)(s+1)/2. */
int aca_get_flip_table(const aca_sim* s, uint64_t* thr, size_t count);
/* Tile grid of the persistent tile kernel: out[0..6] = tiles along x, y, z of one shard,
 * shards on this handle, tile extents x, y, z. ACA_ESTATE for whole-lattice / sync handles. */
int aca_get_tile_grid(const aca_sim* s, int64_t* out);
/* a10 per-tile class bookkeeping (aca_options.class_book = 1, north_star
 * "per-tile Bortz-Kalos-Lebowitz n-fold-way class bookkeeping"): for every tile (shard-major,
 * then (tz * tiles_y + ty) * tiles_x + tx) 16 u32, the number of the tile's cells in BKL class k
 * = (Sigma+z)/2 + (z+1)(s+1)/2 (k < 10 in 2-D, < 14 in 3-D; the rest 0). count = 16 x tiles.
 * refresh = 0: the histograms as the kernels keep them, each tile's classes counted when its
 * last visit wrote it back (a tile whose neighbours fired after that visit may differ from
 * the current state at its boundary cells). refresh = 1: recounted from the current state
 * first (exact; multi-process handles: against the halos of the last run). ACA_ESTATE when
 * class_book is off. Synchronises. */
int aca_get_tile_classes(aca_sim* s, uint32_t* out, size_t count, int refresh);

/* Replace the state from host arrays (checkpoint / resume). Every t must be >= 1 and
 * below the packed-word limit, spins +-1. */
int aca_set_state(aca_sim* s, const int8_t* spins, const uint64_t* times,
                  const uint32_t* counters, size_t count);
/* Replace only the spins (user-supplied initial configuration); times/counters keep
 * their P5 values. */
int aca_set_spins(aca_sim* s, const int8_t* spins, size_t count);

/* Re-initialise (P5) with `seed`: fresh state, counters and statistics, T back to 0.
 * Used to repeat a workload without re-allocating (benchmark steps). Asynchronous. */
int aca_reset(aca_sim* s, uint64_t seed);

void aca_destroy(aca_sim* s);
const char* aca_last_error(void);

/* Multi-process setup: write a fresh 128-byte ncclUniqueId (rank 0 calls this and shares
 * the bytes with the other ranks, e.g. through torch.distributed). NCCL is resolved at run
 * time from the process (the library does not link it); ACA_ENCCL if unavailable. */
int aca_nccl_unique_id(void* out128);

/* Number of cells of the handle (rank-local for multi-process handles). */
int64_t aca_num_cells(const aca_sim* s);

/* ---- Asynchronous spin I/O (pipelining the per-step host copies with the simulation) ----
 * aca_stage_spins: enqueue the host-to-device copy of `count` (= aca_num_cells) spins (+-1, int8,
 *   x fastest) into staging slot `slot` (0 or 1) on the handle's copy stream, and return. The host
 *   buffer must stay valid until the copy is done (aca_sync); pinned memory makes it a DMA.
 * aca_set_spins_staged: the handle's stream waits for that copy, then sets the spins from the
 *   slot (as aca_set_spins: times, counters and ranks unchanged). Returns without waiting.
 * aca_get_spins_async: enqueue the unpacking of the current spins on the handle's stream and
 *   their device-to-host copy into `out` on the copy stream (two output slots alternate);
 *   returns at once. `out` holds the spins of the state at the call after aca_sync.
 * aca_sync: wait for all work enqueued on both streams.
 * Work on the handle's stream stays in call order (reset, set, run_until, getters), so these
 * calls compose with the synchronous API. Staging uses 4 bytes per cell of device memory.
 * Errors: ACA_EINVAL (count, slot, null), ACA_ESTATE (set before any stage), ACA_ENOMEM, ACA_ECUDA. */
int aca_stage_spins(aca_sim* s, const int8_t* spins, size_t count, int slot);
int aca_set_spins_staged(aca_sim* s, int slot);
int aca_get_spins_async(aca_sim* s, int8_t* out, size_t count);
int aca_sync(aca_sim* s);

/* ---- Multi-process push mode (CUDA IPC; world > 1, halo_mode 0) ----
 * One process per GPU owns a strip (2-D) / slab (3-D). Instead of exchanging halos between
 * launches, every rank's tile kernel stores its boundary rows straight into its ring
 * neighbours' halo buffers (over NVLink when they are on other GPUs) as it writes tiles back;
 * a rank never waits for another inside a run (any interleaving is exact: words only grow and
 * are never torn). A run starts with an epoch barrier and ends when every rank reports no
 * active cell, both through small {epoch, active} slots mapped into every process.
 * aca_ipc_export writes this rank's blob (ACA_IPC_BLOB_BYTES: IPC handles of its two halo
 * buffers and its slot); the caller gathers all ranks' blobs in rank order and passes them to
 * aca_ipc_import (world x ACA_IPC_BLOB_BYTES bytes), once, before the first run_until.
 * Errors: ACA_ESTATE (not a push-mode handle / imported twice / run before import), ACA_EINVAL,
 * ACA_ECUDA. Stats, frames and getters are rank-local as for the NCCL mode; the boundary
 * bond term of aca_get_stats reads a snapshot of the neighbours' rows taken when every rank
 * had finished the last run (or their P5 rows after create / reset), so a neighbour's later
 * reset or run does not race with it; after set_state / set_spins a run_until must come first
 * (ACA_ESTATE). Needs the persistent tile kernel (not whole_lattice = 1 or sync_rounds = 1;
 * ACA_EINVAL at create otherwise). */
#define ACA_IPC_BLOB_BYTES 192
int aca_ipc_export(const aca_sim* s, void* out, size_t size);
int aca_ipc_import(aca_sim* s, const void* blobs, size_t size);

/* ---- Output frames (fig:genout) ----
 * Continue the simulation and capture the state of every cell at the frame times
 * K dt, K = K0 .. K0 + count - 1 (the state at time t includes an arrival at exactly t,
 * PAPER.md:355-362). Frames are filled on the device while the cells advance: each fired
 * arrival writes the frames its new state covers. B frames (1..16) are buffered, so the
 * local times of the cells never spread by more than about B dt (the bounded-lag window of
 * PAPER.md:1295-1318); after each window the frames are copied to `out`. On return every
 * arrival at or before (K0 + count - 1) dt has been processed (as aca_run_until_q32 of that
 * time + 1 unit). out: count frames of ceil(N/8) bytes, caller-owned; frame k bit i (byte i/8,
 * bit i%8) = 1 iff cell i (row-major; rank-local for multi-process handles) had s = +1.
 * Errors: ACA_EINVAL (null, dt <= 0, count < 1, B outside 1..16), ACA_ESTATE (K0 dt is
 * before the time already simulated), ACA_ERANGE (frame times overflow), run_until errors. */
int aca_run_frames(aca_sim* s, double dt, int64_t K0, int64_t count, int B, uint8_t* out);

/* ---- Aggregated Poisson stream (fig:amcpoi; docs/PRIMITIVES.md P8) ----
 * The 2-D periodic lattice (dims[0] x dims[1], multiples of m) is partitioned into m x m
 * subarrays (1 <= m <= 32; the paper's experiments use m = 12 and 24, PAPER.md:1476-1488,
 * 1586-1589). Each subarray carries one Poisson stream of rate lambda m^2; at
 * each arrival one of its cells, chosen uniformly at random, is updated (heat-bath or
 * Metropolis, P4), after waiting for the subarrays that hold the cell's outside neighbours.
 * One GPU thread per subarray, conservative launches until every T(C) >= T. The trajectory
 * depends on m; for m = 1 it is the main path's trajectory exactly.
 * Outputs (host, caller-owned, each may be NULL): spins_out[N] (int8 row-major), T_out[ntiles]
 * (Q32 next arrival per subarray), n_out[ntiles] (arrivals per subarray), st. budget: arrivals
 * per subarray per launch (<= 0: 64). Device memory is allocated and freed inside the call.
 * Errors: ACA_EINVAL (arguments), ACA_ENOMEM, ACA_ENODEV, ACA_ECUDA, ACA_ESTATE. */
typedef struct {
    uint64_t arrivals, flips, event_hash;   /* event hash: P7 with the cell choice l mixed in */
    int64_t bond_sum, magnetisation;        /* from spins_out (0 if it is NULL) */
    uint64_t launches;
    double gpu_seconds;                     /* device time of the simulation launches */
} aca_agg_stats;
int aca_agg_run(const int64_t* dims, int m, double lambda, double beta, double J, double h, int rule, uint64_t seed,
                double init_q, double T, int budget, int8_t* spins_out, uint64_t* T_out, uint32_t* n_out,
                aca_agg_stats* st, int device);

/* ---- Modified BKL (docs/PRIMITIVES.md P9) ----
 * Same partition, arguments and outputs as aca_agg_run (2 <= m <= 32; lambda >= 1e-6). In
 * every subarray the boundary layer Gamma_0 (fixed class, weight |Gamma_0|) follows the
 * standard model and waits for the neighbouring subarrays; the (m-2) x (m-2) kernel runs the
 * BKL n-fold way (classes by flip probability, the selected kernel cell always flips), so no
 * state or class change ever crosses a subarray boundary and nothing rolls back. The event
 * counters n(C) count iterations (kernel rejections are skipped); st->flips counts changes. */
int aca_bkl_run(const int64_t* dims, int m, double lambda, double beta, double J, double h, int rule, uint64_t seed,
                double init_q, double T, int budget, int8_t* spins_out, uint64_t* T_out, uint32_t* n_out,
                aca_agg_stats* st, int device);

/* ---- The q-th degree neighbourhood (Eq. nei2 / neiq; docs/PRIMITIVES.md P12) ----
 * The Ising model on neighbors^q(c), the L1 ball of radius q around c (|neighbors^q| - 1 = 2q(q+1)
 * in 2-D): Sigma sums the spins of every member, the P4 table has
 * z = |neighbors^q| - 1 (2 (z + 1) entries), a cell fires only when its (t, c) is below every
 * member's (P6). Draws, increments (law 0..3, P3L; tie_bits P3b), P5 (init_q) and P7 as the main path;
 * q = 1 gives the main path's trajectory. ndim 2 or 3, 1 <= q <= 4, every side >= 2q + 1, N <= 2^32;
 * rounds: synchronous rounds per tile visit (<= 0: 32). Runs from the P5 state to T (fires every
 * arrival t < round-half-up(T 2^32)). Outputs (host, caller-owned, each may be NULL): spins_out[N]
 * int8, t_out[N] Q32 pending times, n_out[N] counters, row-major; st: arrivals, flips, event hash,
 * B (each pair of cells within neighbors^q once), M, launches, sweeps and the device time of the
 * sweeps (initialisation excluded). Device memory (13 N bytes) is allocated and freed inside the
 * call. Errors: ACA_EINVAL (arguments), ACA_ENOMEM, ACA_ENODEV, ACA_ECUDA, ACA_ESTATE. */
typedef struct {
    uint64_t arrivals, flips, event_hash;
    int64_t bond_sum, magnetisation;
    uint64_t launches, sweeps;
    double gpu_seconds;
} aca_qnbr_stats;
int aca_qnbr_run(int ndim, const int64_t* dims, int q, double lambda, double beta, double J, double h, int rule,
                 uint64_t seed, double init_q, int tie_bits, int law, double T, int rounds, int8_t* spins_out,
                 uint64_t* t_out, uint32_t* n_out, aca_qnbr_stats* st, int device);

/* ---- Time-only efficiency model ----
 * Synchronous iterations of fig:s1c1pe on the local times only (valid because next_t does
 * not depend on the states for the Ising model): each iteration every
 * cell whose (t, c) is below all neighbours' (P6 order) draws its next increment of `law`
 * (P3L) at rate lambda. ndim 1 (n-circle), 2 (n x n torus), 3 (periodic n^3); dims[ndim],
 * every dim >= 2. Draws: initial t from Philox ctr (0, c, 0, 1) (P5), iteration r from ctr
 * (r, c_lo, c_hi, 2). Outputs (host buffers, caller-owned): fired_per_round[rounds] = N0 of
 * each iteration (its efficiency is N0/N); t_out[N] (may be NULL) = the
 * final times; *gpu_seconds (may be NULL) = device time of the iterations. device < 0: the
 * current device. Device memory (2 x 8N bytes) is allocated and freed inside the call.
 * Errors: ACA_EINVAL (arguments), ACA_ENOMEM, ACA_ENODEV, ACA_ECUDA. */
int aca_efficiency_run(int ndim, const int64_t* dims, int law, double lambda, uint64_t seed, int64_t rounds,
                       uint64_t* fired_per_round, uint64_t* t_out, int device, double* gpu_seconds);
/* fig:perfbl model (docs/PRIMITIVES.md P11): the simplified many-cells-per-PE model of
 * PAPER.md:1491-1546 (Eq. hC) on a px x py torus of PEs, each carrying an m x m subarray, in the
 * reading where a blocked PE keeps its selected cell (fig:amcpoi Steps 2-3),
 * with the lag bound of fig:perfbl in units of a cell's mean inter-arrival
 * time (lag 0 = unbounded). ups[r] (caller-owned, `rounds` entries) = PEs that advanced in round
 * r; the efficiency (Eq. effi) is their mean over PEs. Optional h_out (u64[px py], Q32) and n_out
 * (u32[px py]): the final state. device < 0: the current device. ACA_EINVAL on bad arguments
 * (1 <= px py <= 2^24, 2 <= m <= 65535), ACA_ENODEV without a GPU. Bit-identical to the
 * oracle's oracle_perfbl_run. */
int aca_perfbl_run(int64_t px, int64_t py, int m, double lag, uint64_t seed, int64_t rounds, uint64_t* ups,
                   uint64_t* h_out, uint32_t* n_out, int device);

/* The same with the q-th degree neighbourhood neighbors^q (Eq. neiq: all
 * cells within Manhattan distance q, |neighbors^q| - 1 = 2q(q+1) on the square array), q in
 * [1, 8]; aca_efficiency_run is q = 1. */
int aca_efficiency_run_q(int ndim, const int64_t* dims, int law, double lambda, uint64_t seed, int64_t rounds, int q,
                         uint64_t* fired_per_round, uint64_t* t_out, int device, double* gpu_seconds);

/* ---- Self-test hooks (device primitives through the ABI; host buffers, n elements) ----
 * P1: out[4n] = our Philox(ctr[4i..], key[2i..]); ref[4n] = cuRAND's device
 *     curand_Philox4x32_10 on the same inputs (library reference for the pin). */
int aca_selftest_philox(uint64_t n, const uint32_t* ctr, const uint32_t* key, uint32_t* out,
                        uint32_t* ref);
/* P3: q[i] = NLOG-2(X[i]); delta[i] = Delta(X[i]) for inv_lambda, tie_bits. */
int aca_selftest_nlog(uint64_t n, const uint64_t* X, uint64_t* q, uint64_t* delta,
                      uint64_t inv_lambda, int tie_bits);
/* P3L: u[i] = unscaled increment of `law` for (w1, w2) = (X[i] >> 32, X[i] & 0xffffffff) (law 4: the
 * period gauss_u(w1, w1, w2, 10) of a cell whose initial draw has w3 = w1 and c_lo = w2);
 * delta[i] = the increment after 1/lambda, the clamp and P3b. ACA_EINVAL for law outside 0..4. */
int aca_selftest_law(uint64_t n, const uint64_t* X, int law, uint64_t inv_lambda, int tie_bits, uint64_t* u,
                     uint64_t* delta);

#ifdef __cplusplus
}
#endif
#endif /* ACA_H */
