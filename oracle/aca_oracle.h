/* aca_oracle.h — serial CPU oracle for the conservative Poisson-asynchronous Ising path.
 *
 * ORACLE / TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (the CUDA package and its shared library) never includes, links or calls it, and this code
 * includes nothing from the product path.
 *
 * What it computes: the plain definition of the trajectory — every arrival processed in
 * increasing lexicographic (t, c) order from a global priority queue (the "standard"
 * serial procedure of PAPER.md:196-211 with per-cell streams, Eq. newt1i),
 * which the conservative parallel algorithms reach exactly (uniqueness argument,
 * PAPER.md:596-613, 833-871, 959-963). Primitives follow docs/PRIMITIVES.md P1-P7.
 */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oracle_sim oracle_sim;

typedef struct {
    uint64_t arrivals, flips, event_hash;
    int64_t bond_sum, magnetisation;
    uint64_t t_min, t_max;
    uint64_t rounds;   /* synchronous-round variant only: rounds executed so far */
} oracle_stats;

/* P1: Philox4x32-10, ctr[4], key[2] -> out[4]. */
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* P3: q = NLOG-2(X) in Q32 (before lambda scaling and the max(1, .) clamp). */
uint64_t oracle_nlog_q32(uint64_t X);
/* P3: Delta(w1, w2) for INV = floor(2^32/lambda + 0.5), tie_bits as P3b. */
uint64_t oracle_delta(uint32_t w1, uint32_t w2, uint64_t inv_lambda, int tie_bits);
uint64_t oracle_inv_lambda(double lambda);
/* P3L: asynchrony laws. law 0 Poisson (= oracle_delta), 1 uniform on (0,1), 2 r^(1/8).
 * oracle_law_q32 is the unscaled increment U in Q32 (before 1/lambda, the clamp and P3b). */
/* P3L laws 3/4: the normal quantile of (w + 1/2) 2^-32, a Gaussian period (mean 1, sd 1/4, Q32) with
 * redraws below one unit, and the fixed period of cell c under law 4. */
double oracle_gauss_z(uint32_t w);
uint64_t oracle_gauss_u(uint32_t w, uint32_t sa, uint32_t sb, uint32_t tag);
uint64_t oracle_cell_period_q32(uint64_t seed, uint64_t c);
uint64_t oracle_law_q32(uint32_t w1, uint32_t w2, int law);
uint64_t oracle_delta_law(uint32_t w1, uint32_t w2, uint64_t inv_lambda, int tie_bits, int law);
/* P4: thresholds, 2*(2*ndim+1) entries written to out; _z: 2*(zc+1) entries for zc neighbours. */
void oracle_flip_table(int ndim, double beta, double J, double h, int rule, uint64_t* out);
void oracle_flip_table_z(int zc, double beta, double J, double h, int rule, uint64_t* out);
/* P7 event hash term: (w3 | 1) * (t ^ (l << 1) ^ [new_spin > 0]) mod 2^64 */
uint64_t oracle_ev_hash(uint32_t w3, uint64_t t, uint64_t l, int new_spin);

/* Returns NULL on invalid arguments. ndim in {2,3}, every dim >= 2, N < 2^32. */
oracle_sim* oracle_create(int ndim, const int64_t* dims, double lambda, double beta, double J,
                          double h, int rule, uint64_t seed, double init_q, int tie_bits);
oracle_sim* oracle_create_law(int ndim, const int64_t* dims, double lambda, double beta, double J,
                              double h, int rule, uint64_t seed, double init_q, int tie_bits, int law);
/* q-th degree neighbourhood (Eq. neiq; docs/PRIMITIVES.md P12): q in [1, 4];
 * q > 1 needs rule 0/1 and every side >= 2q + 1. q = 1 is oracle_create_law. */
oracle_sim* oracle_create_q(int ndim, const int64_t* dims, int q, double lambda, double beta, double J,
                            double h, int rule, uint64_t seed, double init_q, int tie_bits, int law);
/* Eq. neiq applied literally around the origin: writes the offsets of neighbors^q(c) \ {c} to
 * out (at most cap) and returns their number, -1 if more than cap. */
int oracle_q_offsets(int ndim, int q, int (*out)[3], int cap);
/* The cells of neighbors^q(c) \ {c} (with multiplicity for q = 1 on sides of 2) the oracle
 * uses; nb must hold 128 entries. Returns their number. */
int oracle_neighbours(const oracle_sim* s, int64_t c, int64_t* nb);
void oracle_destroy(oracle_sim* s);

/* (A) global priority queue on (t, c): the oracle. Returns 0, or -1 if T decreased. */
int oracle_run_until_q32(oracle_sim* s, uint64_t T_q32);
/* (D) the same queue as (A) organised as a calendar queue (buckets of 2^26 Q32 units, the bucket
 *     in progress a heap on (t, c)): the same event order, bit for bit; faster on large lattices.
 *     Returns 0, -1 if T decreased, -2 on allocation failure. */
int oracle_run_until_calendar(oracle_sim* s, uint64_t T_q32);
/* (B) repeatedly fire a uniformly random eligible local minimum (choice RNG: xorshift64*,
 *     unrelated to Philox). Order-independence invariant. */
int oracle_run_until_random_order(oracle_sim* s, uint64_t T_q32, uint64_t choice_seed);
/* (C) synchronous rounds of fig:s1c1pe: test all, compute privately,
 *     commit. fired_per_round (optional, may be NULL) receives up to max_rounds counts. */
int64_t oracle_run_until_sync(oracle_sim* s, uint64_t T_q32, uint64_t* fired_per_round,
                              int64_t max_rounds);

/* NEGATIVE CONTROL for tests only: synchronous rounds with the bare t <= min rule. */
int64_t oracle_run_until_sync_naive_leq(oracle_sim* s, uint64_t T_q32);

void oracle_get_spins(const oracle_sim* s, int8_t* out);
void oracle_set_spins(oracle_sim* s, const int8_t* spins);
void oracle_get_times(const oracle_sim* s, uint64_t* out);
void oracle_get_counters(const oracle_sim* s, uint32_t* out);
void oracle_get_stats(const oracle_sim* s, oracle_stats* out);
int64_t oracle_num_cells(const oracle_sim* s);

/* Boltzmann-pin helpers on tiny lattices (N <= 20): state code = sum_c [s(c)>0] << c.
 * replicas: hist[code] += 1 for the final state of n_rep independent runs (seed0 + r).
 * time-weighted: one run; weight[code] += time spent in code over (T0, T1] (double). */
int oracle_replica_hist(int ndim, const int64_t* dims, double beta, double J, double h,
                        int rule, uint64_t seed0, int64_t n_rep, uint64_t T_q32,
                        uint64_t* hist);
int oracle_time_weighted_hist(int ndim, const int64_t* dims, double beta, double J, double h,
                              int rule, uint64_t seed, uint64_t T0_q32, uint64_t T1_q32,
                              double* weight);

/* Batch P3, and the per-cell closed form of (t, n) after run_until(T). */
void oracle_nlog_batch(int64_t n, const uint64_t* X, uint64_t* q);
void oracle_cell_time_counter(uint64_t seed, uint64_t c, uint64_t T_q32, uint64_t inv_lambda,
                              int tie_bits, uint64_t* t_out, uint32_t* n_out);
void oracle_cell_time_counter_law(uint64_t seed, uint64_t c, uint64_t T_q32, uint64_t inv_lambda,
                                  int tie_bits, int law, uint64_t* t_out, uint32_t* n_out);

/* Window (light-cone) oracle: exact (s, t, n) of the cell at `center` after run_until(T) on
 * a lattice too large to simulate whole; *exact_out = 0 when the box was too small. */
int oracle_window_cell(int ndim, const int64_t* dims, double lambda, double beta, double J, double h, int rule,
                       uint64_t seed, double init_q, int tie_bits, uint64_t T_q32, const int64_t* center,
                       int64_t radius, int refine, int8_t* s_out, uint64_t* t_out, uint32_t* n_out,
                       int* exact_out);
int oracle_window_cell_law(int ndim, const int64_t* dims, double lambda, double beta, double J, double h, int rule,
                           uint64_t seed, double init_q, int tie_bits, uint64_t T_q32, const int64_t* center,
                           int64_t radius, int refine, int8_t* s_out, uint64_t* t_out, uint32_t* n_out,
                           int* exact_out, int law);

/* fig:perfbl model (docs/PRIMITIVES.md P11): rounds of the simplified many-cells-per-PE model
 * with a lag bound (0 = unbounded). ups[rounds]. */
int oracle_perfbl_run(int64_t px, int64_t py, int m, uint64_t lag_q32, uint64_t seed, int64_t rounds, uint64_t* ups,
                      uint64_t* h_out, uint32_t* n_out);

/* Time-only efficiency model: synchronous iterations on local times,
 * ndim 1..3, law P3L. fired_per_round[rounds] (N0 per iteration) and t_out[N] may be NULL. */
int oracle_efficiency_run(int ndim, const int64_t* dims, int law, double lambda, uint64_t seed, int64_t rounds,
                          uint64_t* fired_per_round, uint64_t* t_out);
/* The same with the q-th degree neighbourhood (Eq. neiq: all cells within Manhattan distance q). */
int oracle_efficiency_run_q(int ndim, const int64_t* dims, int law, double lambda, uint64_t seed, int64_t rounds,
                            int q, uint64_t* fired_per_round, uint64_t* t_out);

/* Aggregated Poisson stream (fig:amcpoi; docs/PRIMITIVES.md P8): 2-D torus
 * in m x m subarrays, one cumulative stream per subarray, serial (T(C), C) order. Outputs may
 * be NULL: spins[N], T[ntiles], n[ntiles]; st gets arrivals, flips, event_hash, B, M. */
int oracle_agg_run(const int64_t* dims, int m, double lambda, double beta, double J, double h, int rule,
                   uint64_t seed, double init_q, uint64_t T_q32, int8_t* spins_out, uint64_t* T_out,
                   uint32_t* n_out, oracle_stats* st);

/* Modified BKL (docs/PRIMITIVES.md P9): per m x m subarray (m = 2, 4, 8)
 * the n-fold way on the kernel, the standard model on the boundary layer; same outputs as
 * oracle_agg_run. */
int oracle_bkl_run(const int64_t* dims, int m, double lambda, double beta, double J, double h, int rule,
                   uint64_t seed, double init_q, uint64_t T_q32, int8_t* spins_out, uint64_t* T_out,
                   uint32_t* n_out, oracle_stats* st);

#ifdef __cplusplus
}
#endif
