// aca_kernels.cuh — sm_100a kernels of the conservative Poisson-asynchronous Ising path.
//
// State in HBM: ONE u64 word per cell (a shard = a run of rows (2-D) / planes (3-D)):
//
//     word = t << TSH | n << 1 | [s(c) = +1]        TSH = NB + 1
//
// t: pending arrival time (Q32), n: event counter (NB bits). A cell's whole state (t, n, s) is
// read and written by one 8-byte access and can never be observed torn. The time occupies the
// top bits, so `word(a) < word(b)` whenever t(a) < t(b): the 32-bit high halves decide the
// (t, c) order of P6 unless they are equal, and only then are the time fields compared and,
// on equal times, the cell ids (lex_lt / id_first below: along an axis the id grows with the
// coordinate except across the periodic wrap). No bits are spent on the tie-break, so the time
// field spans 63 - NB bits and the horizon is not limited by the lattice size. The host chooses
// the (t, n) split per run_until(T) and repacks when T grows; a counter that would overflow its
// field raises ctl->overflow (ACA_ERANGE) instead of wrapping.
//
// In-place updates (no ping-pong): every word a CTA observes for a neighbour is a value that
// neighbour really held, and words only grow. A cell fires only when it precedes every observed
// neighbour; by the stale-read argument of fig:amcgen and the uniqueness
// argument of fig:a1c1pe the neighbour's state at the firing time equals
// the observed one, so any interleaving of CTAs and threads yields the unique trajectory.
#pragma once
#include <stdint.h>

#include <cuda.h>   // CUtensorMap (the tile box of the TMA tensor copies)

#include "aca_prim.cuh"
#include "nlog_tables.cuh"

namespace aca {

// ACA_DEBUG builds (libaca_dbg.so, tests and bug hunts only): device-side invariant checks that
// print the failing condition and trap.
#ifdef ACA_DEBUG
// a failed check records (line, a, b) in the shard's control block (the first one wins) and the
// kernel goes on with the access skipped where possible; the host reports it (ACA_SYNC_DEBUG)
#define ACA_CHECK(cond, a, b)                                                                    \
    do {                                                                                         \
        if (!(cond)) {                                                                           \
            if (atomicCAS(&P.ctl->dbg_line, 0u, (unsigned int)__LINE__) == 0u) {                \
                P.ctl->dbg_a = (unsigned long long)(a);                                          \
                P.ctl->dbg_b = (unsigned long long)(b);                                          \
                if (P.dbg_map) {   /* host-mapped: readable after a fault */                     \
                    P.dbg_map[1] = (unsigned long long)(a);                                      \
                    P.dbg_map[2] = (unsigned long long)(b);                                      \
                    P.dbg_map[3] = blockIdx.x * 1024ull + threadIdx.x;                           \
                    __threadfence_system();                                                      \
                    P.dbg_map[0] = (unsigned long long)__LINE__;                                 \
                    __threadfence_system();                                                      \
                }                                                                                \
            }                                                                                    \
        }                                                                                        \
    } while (0)
#define ACA_DBG_OK(cond) (cond)
// host-mapped trace: lane 0 of every warp records its last stage (survives a kernel fault)
#define ACA_TRACE(code, payload)                                                                 \
    do {                                                                                         \
        if (P.dbg_trace && (threadIdx.x & 31) == 0) {                                            \
            volatile unsigned long long* tr_ = P.dbg_trace + 2 * (blockIdx.x * 32 + (threadIdx.x >> 5)); \
            tr_[1] = ((unsigned long long)(code) << 56) | ((unsigned long long)(payload) & 0xffffffffffffffull); \
            tr_[0] = tr_[0] + 1;                                                                 \
        }                                                                                        \
    } while (0)
#else
#define ACA_TRACE(code, payload) do { } while (0)
#define ACA_CHECK(cond, a, b) do { } while (0)
#define ACA_DBG_OK(cond) true
#endif

struct Ctl {                            // device control block, one per shard
    unsigned long long wlim;            // T_q32 << TSH: fire iff word < wlim  (t < T)
    unsigned long long active_accum;    // cells with t < T after this launch (accumulating)
    unsigned long long active_last;     // value of the last completed launch
    unsigned long long fired, flips, tested, hash;
    unsigned long long launches, inner_rounds;
    unsigned int done;                  // set when a launch ends with no active cell
    unsigned int ticket;                // last-CTA detection
    unsigned int rounds_max;            // max in-tile rounds over CTAs of this launch
    unsigned int overflow;              // an event counter reached its field maximum
    unsigned long long active_carry;    // checkerboard: active cells of the phase-0 tiles
    unsigned int dbg_line, dbg_pad;     // ACA_DEBUG builds: first failed device check
    unsigned long long dbg_a, dbg_b;
    // bounded lag (aca_options.lag): the firing limit wlim of the next launch
    // is min(T, global minimum time + lag); wlim_T keeps T (termination counts cells below it)
    unsigned long long wlim_T;
    unsigned long long wmin[2];         // minimum word of the tiles of each colour at their last write-back
    unsigned long long visits_early, visits_plain;   // a10 class bookkeeping: tile visits per path
    // resident-tile kernel (res_kernel): grid barrier (arrivals, generation) and the active-cell
    // counts of three consecutive sweeps
    unsigned int bar_count, bar_gen;
    unsigned long long res_act[3];
};

struct Geo {
    int ndim;
    int nx, ny, nz;          // local extents (the sharded axis is y in 2-D, z in 3-D)
    int NY, NZ;              // global extents of y and z
    int y0, z0;              // global offset of the shard along the sharded axis
    int sharded;             // 0: periodic wrap inside the storage; 1: halo buffers
    int NB, TSH;             // counter bits, time shift (= NB + 1)
    unsigned int nbmask;     // (1 << NB) - 1: the counter field's mask and its saturated value
};

__device__ __host__ __forceinline__ unsigned long long w_time(unsigned long long w, const Geo& g) { return w >> g.TSH; }
__device__ __host__ __forceinline__ unsigned int w_count(unsigned long long w, const Geo& g) {
    return (unsigned int)(w >> 1) & g.nbmask;   // NB <= 31
}
__device__ __host__ __forceinline__ unsigned long long w_pack(unsigned long long t, unsigned long long n,
                                                              unsigned long long sb, const Geo& g) {
    return (t << g.TSH) | (n << 1) | sb;
}
__device__ __forceinline__ unsigned int hi32(unsigned long long w) { return (unsigned int)(w >> 32); }

// P6 on the rank-free words. id_first(q): does cell c (global coordinates gx, gy, gz) come
// before its neighbour in direction q (0: -x, 1: +x, 2: -y, 3: +y, 4: -z, 5: +z) in the
// row-major id order (c = y nx + x, c = (z NY + y) nx + x)? Along an axis the id grows with the
// coordinate, except across the periodic wrap; a side of length 2 makes both neighbours the
// same cell and the rule gives the same answer for both. lex_lt(a, b, a_first): is (t(a), a)
// below (t(b), b)?
__device__ __forceinline__ bool id_first(const Geo& g, int q, int gx, int gy, int gz) {
    switch (q) {
        case 0: return gx == 0;
        case 1: return gx < g.nx - 1;
        case 2: return gy == 0;
        case 3: return gy < g.NY - 1;
        case 4: return gz == 0;
        default: return gz < g.NZ - 1;
    }
}
__device__ __forceinline__ bool lex_lt(unsigned long long a, unsigned long long b, int TSH, bool a_first) {
    const unsigned long long ta = a >> TSH, tb = b >> TSH;
    return ta < tb || (ta == tb && a_first);
}

// Output frames (fig:genout): the state of every cell at the frame times
// tau_k = t0 + k dt, k = 0..nb-1, one bit per cell (+1 = 1) in frame k of `bits` (words of
// `wpf` u32 each). A fired arrival at t_p (new spin s', next arrival t_n) owns the frames with
// t_p <= tau_k < t_n: s' is the cell's state on [t_p, t_n) ("at time t the value is already
// new"). Frames before the first arrival of a chunk are pre-filled on the
// host side (frame_prefill_kernel).
struct FrameParams {
    unsigned int* bits;
    unsigned long long t0, dt;           // Q32
    unsigned long long wpf;              // u32 words per frame
    long long base;                      // cell id of bit 0 (rank-local frames)
    int nb;                              // frames in the window (0 = off)
};

__device__ __forceinline__ void frame_write(const FrameParams& F, unsigned long long tp, unsigned long long tn,
                                            unsigned long long c, uint32_t splus) {
    if (F.nb == 0 || !splus || tn <= F.t0) return;
    const unsigned long long b = c - (unsigned long long)F.base;
    unsigned long long tau = F.t0;
    for (int k = 0; k < F.nb; ++k, tau += F.dt) {
        if (tau >= tn) break;
        if (tau >= tp) atomicOr(F.bits + (size_t)k * F.wpf + (b >> 5), 1u << (b & 31));
    }
}

struct KParams {
    // TMA tensor map of the shard's words (2-D [ny][nx] / 3-D [nz][ny][nx] u64, box = a tile with
    // its 2-word x halo and 1-cell y (z) halo); tile_grp_kernel stages interior tiles with ONE
    // cp.async.bulk.tensor per tile. Zeroed (box_ok = 0) when the host could not encode it.
    CUtensorMap tmap;
    int box_ok;
    Geo g;
    unsigned long long* words;
    const unsigned long long* halo_lo;   // sharded axis: row/plane just below the shard
    const unsigned long long* halo_hi;   // ... and just above
    // push mode (sharded): where this shard's first / last row (plane) goes — the lower
    // neighbour's halo_hi and the upper neighbour's halo_lo (same device, or a peer GPU's memory
    // mapped over NVLink). nullptr: halos are exchanged between launches instead.
    unsigned long long* push_lo;
    unsigned long long* push_hi;
    Ctl* ctl;
    const unsigned long long* lr;        // device copy of ACA_NLOG_LR (512 entries)
    uint32_t key0, key1;
    uint32_t rk[20];                     // Philox round keys of (key0, key1)
    unsigned long long inv_lambda;
    int tie_bits;
    int law;                             // P3L asynchrony law (0 Poisson, 1 uniform, 2 r^(1/8), 3 Gaussian)
    int rounds;                          // R_max
    int do_hash;
    int early;                           // a10: queue early-rejection candidates
    int bulk;                            // max arrivals committed per cell per fire step (1 = one)
    int halo_peer;                       // the halo buffers are written concurrently by peer processes
    int tiles_x, tiles_y, tiles_z;
    int phase;                           // -1: every tile; 0 / 1: tiles of that checkerboard colour
    int row_par0;                        // parity of the shard's first tile row (global colouring)
    unsigned long long thr[14];          // P4 table
    unsigned long long thm[98];          // a10 table, see commit_loop (2 (Z+1)^2 entries)
    FrameParams fr;                      // output frames (off unless aca_run_frames)
    int fast;                            // fire_fast applies (law 0, lambda 1, no ties, no frames, N < 2^32)
    int life;                            // rule 2: asynchronous Game of Life (Moore neighbourhood, P10)
    unsigned long long lag_q;            // bounded lag in Q32 (0 = off)
    // a10 per-tile class bookkeeping (tile_grp_kernel EM = 2): 16 u32 per tile (BKL classes in the
    // P4 index), the class weights floor(p_k 2^16) and the early-path limit on sum_k |Gamma_k| w_k
    unsigned int* tile_hist;
    unsigned int clsw[16];
    long long cls_lim;
    unsigned long long* dbg_trace;       // ACA_DEBUG: host-mapped stage trace (nullptr = off)
    unsigned long long* dbg_map;         // ACA_DEBUG: host-mapped record of the first failed check
};

__device__ __forceinline__ int wrapi(int v, int n) {
    v %= n;
    return v < 0 ? v + n : v;
}
// v in [-n, 2n): one conditional add/sub instead of an integer division
__device__ __forceinline__ int wrap1(int v, int n) { return v < 0 ? v + n : (v >= n ? v - n : v); }

// An 8-byte word another CTA, GPU or process may be storing concurrently: a relaxed load is a
// single-copy-atomic 8-byte access (PTX memory model), so it returns a state the cell really
// held — never a torn mix of an old time and a new spin.
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Address of the word at (gx, gy, gz) (periodic wrap inside the storage, or the shard's halo
// buffers along the sharded axis). ONE: the coordinates are at most one period out of range.
template <bool ONE>
__device__ __forceinline__ const unsigned long long* word_ptr_t(const KParams& P, int gx, int gy, int gz) {
    const Geo& g = P.g;
    const int x = ONE ? wrap1(gx, g.nx) : wrapi(gx, g.nx);
    if (g.ndim == 2) {
        if (!g.sharded) return P.words + (size_t)(ONE ? wrap1(gy, g.ny) : wrapi(gy, g.ny)) * g.nx + x;
        if (gy < 0) return P.halo_lo + x;
        if (gy >= g.ny) return P.halo_hi + x;
        return P.words + (size_t)gy * g.nx + x;
    }
    const int y = ONE ? wrap1(gy, g.ny) : wrapi(gy, g.ny);
    if (!g.sharded) return P.words + ((size_t)(ONE ? wrap1(gz, g.nz) : wrapi(gz, g.nz)) * g.ny + y) * g.nx + x;
    if (gz < 0) return P.halo_lo + (size_t)y * g.nx + x;
    if (gz >= g.nz) return P.halo_hi + (size_t)y * g.nx + x;
    return P.words + ((size_t)gz * g.ny + y) * g.nx + x;
}
template <bool ONE>
__device__ __forceinline__ unsigned long long ld_word_t(const KParams& P, int gx, int gy, int gz) {
    return ld_relaxed(word_ptr_t<ONE>(P, gx, gy, gz));
}
__device__ __forceinline__ unsigned long long ld_word(const KParams& P, int gx, int gy, int gz) {
    return ld_word_t<false>(P, gx, gy, gz);
}

// Write-back of one owned word; in push mode a word of the shard's first / last row (plane) is
// also stored into the neighbour shard's halo. Any interleaving with the neighbour's reads is
// exact: an aligned 8-byte word is never torn, every stored value is a state the cell really
// held and words only grow (stale-read argument of fig:amcgen), so the
// neighbour needs no synchronisation with this store — it sees an older or a newer state.
__device__ __forceinline__ void push_word(const KParams& P, int gx, int gy, int gz, unsigned long long w) {
    const Geo& g = P.g;
    if (!P.push_lo) return;
    const int a = g.ndim == 2 ? gy : gz, n = g.ndim == 2 ? g.ny : g.nz;
    const size_t f = g.ndim == 2 ? (size_t)gx : (size_t)gy * g.nx + gx;
    if (a == 0) P.push_lo[f] = w;
    if (a == n - 1) P.push_hi[f] = w;
}

// ---------------------------------------------------------------- TMA bulk-copy helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// one 16-B aligned pair of shared words, read as a volatile (each 8-B word single-copy atomic)
__device__ __forceinline__ ulonglong2 lds128v(const volatile unsigned long long* p) {
    ulonglong2 v;
    asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "r"(smem_u32((const void*)p)) : "memory");
    return v;
}
// the same through a 32-bit shared-window address
__device__ __forceinline__ ulonglong2 lds128a(uint32_t a) {
    ulonglong2 v;
    asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ unsigned int lds32a(uint32_t a) {
    unsigned int v;
    asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}"
                 ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// announce `bytes` of async-proxy transfers for the current phase without arriving
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}"
        ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// global -> shared bulk copy (size % 16 == 0, both addresses 16-B aligned), completes on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s_a(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
// the tile box at (x, y[, z]) of the tensor map -> shared memory (128-B aligned), completes on bar
__device__ __forceinline__ void tma_box_2d(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t bar) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(dst), "l"(map), "r"(x), "r"(y), "r"(bar) : "memory");
}
__device__ __forceinline__ void tma_box_3d(uint32_t dst, const CUtensorMap* map, int x, int y, int z, uint32_t bar) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(dst), "l"(map), "r"(x), "r"(y), "r"(z), "r"(bar) : "memory");
}
// order earlier generic-proxy accesses of shared memory before later async-proxy (TMA) ones
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// named barrier of one thread group (ids 1..15; id 0 is __syncthreads)
__device__ __forceinline__ void group_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Block-wide sum (result valid in thread 0).
template <int NT>
__device__ __forceinline__ unsigned long long block_sum(unsigned long long v, unsigned long long* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    unsigned long long s = 0;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) s += red[w];
    }
    return s;
}

// One arrival of a cell (fig:a1c1pe steps 3-4; Appendix).
// `ones` = number of +1 neighbours (with multiplicity), z = coordination number. Returns
// ok = false (and raises ctl->overflow) when the counter field is full.
struct FireOut { unsigned long long wnew; uint32_t flip; unsigned long long h; bool ok; };

template <class Tab>
__device__ __forceinline__ FireOut fire(unsigned long long w, uint32_t ones, int z, unsigned long long c,
                                        const Geo& g, const unsigned long long* thr, const Tab& tab,
                                        const uint32_t* rk, unsigned long long inv_lambda, int tie_bits,
                                        int do_hash, Ctl* ctl, int law = 0, const FrameParams* fr = nullptr) {
    FireOut o;
    const uint32_t k = w_count(w, g);
    if (k == g.nbmask) {
        atomicOr(&ctl->overflow, 1u);
        o.wnew = w; o.flip = 0; o.h = 0; o.ok = false;
        return o;
    }
    const uint32_t sb = (uint32_t)(w & 1ull);
    const uint32_t idx = ones + (uint32_t)(z + 1) * sb;          // (Sigma+z)/2 + (z+1)(s+1)/2
    const u32x4 r = philox4x32_10_rk(k, (uint32_t)c, (uint32_t)(c >> 32), 0u, rk);
    // z = 8: asynchronous Game of Life (P10), Conway's rule on the Moore neighbourhood
    const uint32_t flip = z == 8 ? ((ones == 3u || (sb && ones == 2u)) ? 1u : 0u) ^ sb
                                 : ((unsigned long long)r.x < thr[idx] ? 1u : 0u);
    const unsigned long long d = delta_cell_t(c, rk, r.y, r.z, tab, ACA_LN2_Q48, inv_lambda, tie_bits, law);
    o.wnew = (w + (d << g.TSH) + 2ull) ^ (unsigned long long)flip;   // t += d, n += 1, s ^= flip
    o.flip = flip;
    if (fr && fr->nb) {
        const unsigned long long tp = w >> g.TSH;
        frame_write(*fr, tp, tp + d, c, sb ^ flip);
    }
    o.h = 0;
    o.ok = true;
    if (do_hash) o.h = ev_hash(r.w, w >> g.TSH, (unsigned long long)(sb ^ flip));
    return o;
}

// Last-CTA bookkeeping of one launch: publish counters, decide termination.
// Checkerboard phases: a sweep is two launches (phase 0, then phase 1); the phase-0 tiles do
// not change during phase 1, so their active count carries over and the sweep ends (and
// termination is decided) with phase 1.
__device__ __forceinline__ void finish_launch(Ctl* ctl, unsigned long long active, unsigned long long fired,
                                              unsigned long long flips, unsigned long long tested,
                                              unsigned long long hash, unsigned int rounds, int phase = -1,
                                              unsigned long long lag_q = 0, int tsh = 0) {
    atomicAdd(&ctl->active_accum, active);
    if (fired) atomicAdd(&ctl->fired, fired);
    if (flips) atomicAdd(&ctl->flips, flips);
    if (tested) atomicAdd(&ctl->tested, tested);
    if (hash) atomicAdd(&ctl->hash, hash);
    atomicMax(&ctl->rounds_max, rounds);
    __threadfence();
    const unsigned int ticket = atomicAdd(&ctl->ticket, 1u);
    if (ticket == gridDim.x * gridDim.y * gridDim.z - 1) {
        __threadfence();
        unsigned long long act = atomicAdd(&ctl->active_accum, 0ull);
        ctl->inner_rounds += atomicAdd(&ctl->rounds_max, 0u);
        ctl->active_accum = 0ull;
        if (phase == 0) {
            ctl->active_carry = act;
        } else {
            if (phase == 1) act += ctl->active_carry;
            ctl->active_last = act;
            ctl->done = (act == 0ull || ctl->overflow) ? 1u : 0u;
            ctl->launches += 1ull;
        }
        ctl->rounds_max = 0u;
        if (lag_q) {   // next launch: fire only below (global minimum time + lag), and below T
            const int q = phase < 0 ? 0 : phase;
            const unsigned long long wm = phase < 0 ? ctl->wmin[0] : min(ctl->wmin[0], ctl->wmin[1]);
            const unsigned long long tl = (wm >> tsh) + lag_q;
            const unsigned long long wl = tl < (ctl->wlim_T >> tsh) ? tl << tsh : ctl->wlim_T;
            ctl->wlim = wl;
            ctl->wmin[phase < 0 ? 0 : 1 - q] = ~0ull;   // recomputed by the launch that comes next
        }
        __threadfence();
        ctl->ticket = 0u;
    }
}

__device__ __forceinline__ unsigned long long cell_id(const Geo& g, int gx, int gy, int gz) {
    return g.ndim == 2 ? (unsigned long long)(gy + g.y0) * g.nx + gx
                       : ((unsigned long long)(gz + g.z0) * g.NY + gy) * g.nx + gx;
}
// 32-bit cell id (N < 2^32; the Philox counter word c_hi is then 0)
template <int NDIM>
__device__ __forceinline__ uint32_t cell_id32t(const Geo& g, int gx, int gy, int gz) {
    return NDIM == 2 ? (uint32_t)(gy + g.y0) * (uint32_t)g.nx + (uint32_t)gx
                     : ((uint32_t)(gz + g.z0) * (uint32_t)g.NY + (uint32_t)gy) * (uint32_t)g.nx + (uint32_t)gx;
}

// fire() for the common configuration (Poisson law, lambda = 1, tie_bits = 0, no output frames,
// N < 2^32): the same integers with the general branches compiled out; the P4 table is read
// through its shared-window address `thr_a`. The caller raises the overflow flag when ok = false.
__device__ __forceinline__ FireOut fire_fast(unsigned long long w, uint32_t ones, int z, uint32_t c, const Geo& g,
                                             uint32_t thr_a, const NlogSmem& tab, const uint32_t* rk, int do_hash) {
    FireOut o;
    const uint32_t k = w_count(w, g);
    o.ok = k != g.nbmask;
    const uint32_t sb = (uint32_t)(w & 1ull);
    const uint32_t idx = ones + (uint32_t)(z + 1) * sb;
    const u32x4 r = philox4x32_10_rk(k, c, 0u, 0u, rk);
    uint32_t flip;
    if (z == 8) {
        flip = ((ones == 3u || (sb && ones == 2u)) ? 1u : 0u) ^ sb;
    } else {
        unsigned long long t;
        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(t) : "r"(thr_a + 8u * idx));
        flip = (unsigned long long)r.x < t ? 1u : 0u;
    }
    uint64_t d = nlog_q32_t(((uint64_t)r.y << 32) | r.z, tab, ACA_LN2_Q48);
    d = d < 1ull ? 1ull : d;
    o.wnew = (w + (d << g.TSH) + 2ull) ^ (unsigned long long)flip;
    o.flip = flip;
    o.h = 0;
    if (do_hash) o.h = ev_hash(r.w, w >> g.TSH, (unsigned long long)(sb ^ flip));
    return o;
}

// High-half tests of two horizontally adjacent cells (PAIRMAP; the same for one cell, COLMAP).
// Cell k (k = 0, 1) is active iff ah_k < wh, a candidate iff also ah_k <= m_k (m_k = minimum of
// its neighbours' high halves): bit `bit0 << k` of em. Any equality (ah_k == m_k, or ah_k == wh
// when the horizon's low half is not 0) clears `tie`, sending the lane to the exact pass.
// Written with explicit predicates so each decision is one compare and one predicated op.
// The _strict forms decide on strict inequalities only (active iff ah < wh, eligible iff
// ah < m, which is exact: a strictly lower high half is a lower time) and defer the tied
// cells to the next exact round; they count no ties.
__device__ __forceinline__ void one_test(unsigned int ah, unsigned int m, unsigned int wh, uint32_t bit, uint32_t& em,
                                         int& nt, unsigned int& tie) {
    asm("{\n\t.reg .pred pa, pl, pt;\n\t"
        "setp.lt.u32 pa, %3, %5;\n\t"
        "setp.le.and.u32 pl, %3, %4, pa;\n\t"
        "@pl or.b32 %0, %0, %6;\n\t"
        "@pa add.s32 %1, %1, 1;\n\t"
        "setp.eq.u32 pt, %3, %4;\n\t"
        "setp.eq.or.u32 pt, %3, %5, pt;\n\t"
        "@pt mov.u32 %2, 0;\n\t}"
        : "+r"(em), "+r"(nt), "+r"(tie)
        : "r"(ah), "r"(m), "r"(wh), "r"(bit));
}
__device__ __forceinline__ void one_test_m(unsigned int ah, unsigned int m, unsigned int wh, uint32_t bit, uint32_t& em,
                                           int& nt, unsigned int& tie) {
    asm("{\n\t.reg .pred pa, pl, pt;\n\t"
        "setp.lt.u32 pa, %3, %5;\n\t"
        "setp.le.and.u32 pl, %3, %4, pa;\n\t"
        "@pl or.b32 %0, %0, %6;\n\t"
        "@pa add.s32 %1, %1, 1;\n\t"
        "setp.eq.u32 pt, %3, %4;\n\t"
        "@pt mov.u32 %2, 0;\n\t}"
        : "+r"(em), "+r"(nt), "+r"(tie)
        : "r"(ah), "r"(m), "r"(wh), "r"(bit));
}
__device__ __forceinline__ void one_test_strict(unsigned int ah, unsigned int m, unsigned int wh, uint32_t bit,
                                                uint32_t& em, int& nt) {
    asm("{\n\t.reg .pred pa, pl;\n\t"
        "setp.lt.u32 pa, %2, %4;\n\t"
        "setp.lt.and.u32 pl, %2, %3, pa;\n\t"
        "@pl or.b32 %0, %0, %5;\n\t"
        "@pa add.s32 %1, %1, 1;\n\t}"
        : "+r"(em), "+r"(nt)
        : "r"(ah), "r"(m), "r"(wh), "r"(bit));
}
__device__ __forceinline__ void pair_test(unsigned int ah0, unsigned int ah1, unsigned int m0, unsigned int m1,
                                          unsigned int wh, uint32_t bit0, uint32_t& em, int& nt,
                                          unsigned int& tie) {
    asm("{\n\t.reg .pred pa, pb, pl, pm, pt;\n\t"
        "setp.lt.u32 pa, %3, %7;\n\t"
        "setp.lt.u32 pb, %4, %7;\n\t"
        "setp.le.and.u32 pl, %3, %5, pa;\n\t"
        "setp.le.and.u32 pm, %4, %6, pb;\n\t"
        "@pl or.b32 %0, %0, %8;\n\t"
        "@pm or.b32 %0, %0, %9;\n\t"
        "@pa add.s32 %1, %1, 1;\n\t"
        "@pb add.s32 %1, %1, 1;\n\t"
        "setp.eq.u32 pt, %3, %5;\n\t"
        "setp.eq.or.u32 pt, %4, %6, pt;\n\t"
        "setp.eq.or.u32 pt, %3, %7, pt;\n\t"
        "setp.eq.or.u32 pt, %4, %7, pt;\n\t"
        "@pt mov.u32 %2, 0;\n\t}"
        : "+r"(em), "+r"(nt), "+r"(tie)
        : "r"(ah0), "r"(ah1), "r"(m0), "r"(m1), "r"(wh), "r"(bit0), "r"(bit0 << 1));
}
// exact round when wlim's low half is 0: high(w) < high(wlim) <=> w < wlim, no horizon tie
__device__ __forceinline__ void pair_test_m(unsigned int ah0, unsigned int ah1, unsigned int m0, unsigned int m1,
                                            unsigned int wh, uint32_t bit0, uint32_t& em, int& nt, unsigned int& tie) {
    asm("{\n\t.reg .pred pa, pb, pl, pm, pt;\n\t"
        "setp.lt.u32 pa, %3, %7;\n\t"
        "setp.lt.u32 pb, %4, %7;\n\t"
        "setp.le.and.u32 pl, %3, %5, pa;\n\t"
        "setp.le.and.u32 pm, %4, %6, pb;\n\t"
        "@pl or.b32 %0, %0, %8;\n\t"
        "@pm or.b32 %0, %0, %9;\n\t"
        "@pa add.s32 %1, %1, 1;\n\t"
        "@pb add.s32 %1, %1, 1;\n\t"
        "setp.eq.u32 pt, %3, %5;\n\t"
        "setp.eq.or.u32 pt, %4, %6, pt;\n\t"
        "@pt mov.u32 %2, 0;\n\t}"
        : "+r"(em), "+r"(nt), "+r"(tie)
        : "r"(ah0), "r"(ah1), "r"(m0), "r"(m1), "r"(wh), "r"(bit0), "r"(bit0 << 1));
}
__device__ __forceinline__ void pair_test_strict(unsigned int ah0, unsigned int ah1, unsigned int m0, unsigned int m1,
                                                 unsigned int wh, uint32_t bit0, uint32_t& em, int& nt) {
    asm("{\n\t.reg .pred pa, pb, pl, pm;\n\t"
        "setp.lt.u32 pa, %2, %6;\n\t"
        "setp.lt.u32 pb, %3, %6;\n\t"
        "setp.lt.and.u32 pl, %2, %4, pa;\n\t"
        "setp.lt.and.u32 pm, %3, %5, pb;\n\t"
        "@pl or.b32 %0, %0, %7;\n\t"
        "@pm or.b32 %0, %0, %8;\n\t"
        "@pa add.s32 %1, %1, 1;\n\t"
        "@pb add.s32 %1, %1, 1;\n\t}"
        : "+r"(em), "+r"(nt)
        : "r"(ah0), "r"(ah1), "r"(m0), "r"(m1), "r"(wh), "r"(bit0), "r"(bit0 << 1));
}

// Exact P6 test of the cell in slot s (word w, global coordinates gx, gy, gz) against its
// neighbours in shared memory: the von Neumann neighbourhood, or (MOORE) the 8 cells of the
// Moore neighbourhood, whose diagonal neighbours sit in another row, so the row decides.
template <int NDIM, bool MOORE, int SX, int SXY>
__device__ __forceinline__ bool exact_min(const volatile unsigned long long* VS, int s, unsigned long long w,
                                          const Geo& g, int gx, int gy, int gz) {
    const int off[6] = {-1, 1, -SX, SX, -SXY, SXY};
    bool e = true;
#pragma unroll
    for (int q = 0; q < 2 * NDIM; ++q) e = e && lex_lt(w, VS[s + off[q]], g.TSH, id_first(g, q, gx, gy, gz));
    if (MOORE) {
#pragma unroll
        for (int dy = -1; dy <= 1; dy += 2)
#pragma unroll
            for (int dx = -1; dx <= 1; dx += 2)
                e = e && lex_lt(w, VS[s + dy * SX + dx], g.TSH, id_first(g, dy < 0 ? 2 : 3, gx, gy, gz));
    }
    return e;
}
// a10: u = neighbours before the cell in (t, c) order (those that may still change before its
// arrival), k = +1 spins among the others; exact.
template <int NDIM, int SX, int SXY>
__device__ __forceinline__ void early_uk(const volatile unsigned long long* VS, int s, unsigned long long w,
                                         const Geo& g, int gx, int gy, int gz, uint32_t& u, uint32_t& k) {
    const int off[6] = {-1, 1, -SX, SX, -SXY, SXY};
    u = 0;
    k = 0;
#pragma unroll
    for (int q = 0; q < 2 * NDIM; ++q) {
        const unsigned long long nb = VS[s + off[q]];
        const bool below = lex_lt(nb, w, g.TSH, !id_first(g, q, gx, gy, gz));
        u += below;
        k += below ? 0u : (uint32_t)(nb & 1ull);
    }
}

// ------------------------------------------------------------------------ synchronous rounds
// fig:s1c1pe inside a tile (sync_rounds = 1): one CTA per tile, the tile plus a one-cell halo
// staged in shared memory, up to R rounds of the two barriers of fig:s1c1pe:
// every cell decides on one snapshot and keeps its new word private, then all commit. This is
// the exact synchronous round whose firing fraction N0/N is the paper's efficiency
// (PAPER.md:1337-1353); a reference kernel, not the production path.
template <int NDIM, int TX, int TY, int TZ, int NT>
__global__ void __launch_bounds__(NT) tile_sync_kernel(const KParams P) {
    constexpr int SX = TX + 2, SY = TY + 2, SZ = (NDIM == 3) ? TZ + 2 : 1;
    constexpr int NSLOT = SX * SY * SZ;
    constexpr int NCELL = TX * TY * TZ;
    constexpr int CPT = NCELL / NT;
    static_assert(NCELL % NT == 0, "tile must be a multiple of the block");
    constexpr int Z = 2 * NDIM;
    constexpr int SXY = SX * SY;

    if (*(volatile unsigned int*)&P.ctl->done) return;

    extern __shared__ __align__(128) unsigned long long smem[];
    unsigned long long* S = smem;                     // NSLOT words
    unsigned long long* lr = S + NSLOT;               // 512
    unsigned long long* thr = lr + 512;               // 16
    unsigned long long* red = thr + 16;               // NT/32

    const Geo& g = P.g;
    const int tid = threadIdx.x;
    const int bt = blockIdx.x;
    const int tx = bt % P.tiles_x;
    const int ty = (bt / P.tiles_x) % P.tiles_y;
    const int tz = bt / (P.tiles_x * P.tiles_y);
    const int x0 = tx * TX, y0 = ty * TY, z0 = tz * TZ;

    for (int i = tid; i < 512; i += NT) lr[i] = P.lr[i];
    if (tid < 16) thr[tid] = tid < 14 ? P.thr[tid] : 0ull;
    for (int i = tid; i < NSLOT; i += NT) {
        const int lx = i % SX - 1, ly = (i / SX) % SY - 1, lz = (NDIM == 3) ? i / SXY - 1 : 0;
        const int out = (lx < 0 || lx >= TX) + (ly < 0 || ly >= TY) + ((NDIM == 3) && (lz < 0 || lz >= TZ));
        if (out <= 1) S[i] = ld_word(P, x0 + lx, y0 + ly, z0 + lz);
    }
    const NlogLR tab{lr};

    unsigned long long wreg[CPT];
    uint32_t valid = 0;
    const unsigned long long wlim = *(volatile unsigned long long*)&P.ctl->wlim;
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        const int i = tid + k * NT;
        const int lx = i % TX, ly = (i / TX) % TY, lz = i / (TX * TY);
        if (x0 + lx < g.nx && y0 + ly < g.ny && (NDIM == 2 || z0 + lz < g.nz)) valid |= 1u << k;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        const int i = tid + k * NT;
        const int lx = i % TX, ly = (i / TX) % TY, lz = i / (TX * TY);
        wreg[k] = S[(lz + (NDIM == 3)) * SXY + (ly + 1) * SX + lx + 1];
    }
    uint32_t changed = 0;
    volatile unsigned long long* VS = S;

    unsigned long long fired = 0, flips = 0, tested = 0, hacc = 0;
    unsigned int rounds = 0;
    for (int r = 0; r < P.rounds; ++r) {
        int any = 0;
        unsigned long long pend[CPT];
        uint32_t pmask = 0;
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            if (!((valid >> k) & 1u)) continue;
            const unsigned long long w = wreg[k];
            if (w >= wlim) continue;
            ++tested;
            const int i = tid + k * NT;
            const int lx = i % TX, ly = (i / TX) % TY, lz = i / (TX * TY);
            const int s = (lz + (NDIM == 3)) * SXY + (ly + 1) * SX + lx + 1;
            const int gx = x0 + lx, gy = y0 + ly + (NDIM == 2 ? g.y0 : 0), gz = z0 + lz + (NDIM == 3 ? g.z0 : 0);
            if (!exact_min<NDIM, false, SX, SXY>(VS, s, w, g, gx, gy, gz)) continue;
            uint32_t ones = (uint32_t)(VS[s - 1] & 1ull) + (uint32_t)(VS[s + 1] & 1ull) +
                            (uint32_t)(VS[s - SX] & 1ull) + (uint32_t)(VS[s + SX] & 1ull);
            if (NDIM == 3) ones += (uint32_t)(VS[s - SXY] & 1ull) + (uint32_t)(VS[s + SXY] & 1ull);
            const FireOut o = fire(w, ones, Z, cell_id(g, x0 + lx, y0 + ly, z0 + lz), g, thr, tab, P.rk,
                                   P.inv_lambda, P.tie_bits, P.do_hash, P.ctl, P.law, &P.fr);
            if (!o.ok) continue;
            hacc += o.h;
            flips += o.flip;
            ++fired;
            changed |= 1u << k;
            any = 1;
            pend[k] = o.wnew;
            pmask |= 1u << k;
        }
        __syncthreads();                                   // barrier 1 of fig:s1c1pe
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            if ((pmask >> k) & 1u) {
                const int i = tid + k * NT;
                const int lx = i % TX, ly = (i / TX) % TY, lz = i / (TX * TY);
                const int s = (lz + (NDIM == 3)) * SXY + (ly + 1) * SX + lx + 1;
                wreg[k] = pend[k];
                VS[s] = wreg[k];
            }
        }
        ++rounds;
        if (__syncthreads_count(any) == 0) break;              // barrier 2 / stall detection
    }

    unsigned long long active = 0;
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        if (!((valid >> k) & 1u)) continue;
        const int i = tid + k * NT;
        const int lx = i % TX, ly = (i / TX) % TY, lz = i / (TX * TY);
        const int gx = x0 + lx, gy = y0 + ly, gz = z0 + lz;
        const size_t gi = NDIM == 2 ? (size_t)gy * g.nx + gx : ((size_t)gz * g.ny + gy) * g.nx + gx;
        if ((changed >> k) & 1u) {
            P.words[gi] = wreg[k];
            push_word(P, gx, gy, gz, wreg[k]);
        }
        active += wreg[k] < wlim;
    }
    const unsigned long long s_act = block_sum<NT>(active, red);
    const unsigned long long s_fir = block_sum<NT>(fired, red);
    const unsigned long long s_flp = block_sum<NT>(flips, red);
    const unsigned long long s_tst = block_sum<NT>(tested, red);
    const unsigned long long s_hsh = block_sum<NT>(hacc, red);
    if (tid == 0) finish_launch(P.ctl, s_act, s_fir, s_flp, s_tst, s_hsh, rounds);
}
__host__ __device__ constexpr size_t sync_smem_bytes(int ndim, int tx, int ty, int tz, int nt) {
    return ((size_t)(tx + 2) * (ty + 2) * (ndim == 3 ? tz + 2 : 1) + 512 + 16 + nt / 32) * 8;
}

#include "aca_tile.cuh"

#include "aca_res.cuh"

#include "aca_misc.cuh"

}  // namespace aca
