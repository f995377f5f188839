// aca_kernels.cuh — sm_100a kernels of the conservative Poisson-asynchronous Ising path.
//
// State in HBM: ONE u64 word per cell (a shard = a run of rows (2-D) / planes (3-D)):
//
//     word = t << TSH | rank(c) << (NB + 1) | n << 1 | [s(c) = +1]        TSH = RB + NB + 1
//
// t: pending arrival time (Q32), n: event counter (NB bits), rank(c) = x + y (+ z) in global
// coordinates (RB bits). For every neighbour pair rank orders the two cells exactly as their
// row-major ids do (along an axis the id grows with the coordinate, and the periodic pair
// (n-1, 0) is ordered the same way by both), and ranks of neighbours always differ, so the
// bits below the rank never decide a comparison: one unsigned 64-bit compare
// `word(c) < word(c')` is the lexicographic (t, c) test of P6. A cell's whole state
// (t, n, s) is read and written by one 8-byte access and can never be observed torn.
// The host chooses the (t, n) split per run_until(T) and repacks when T grows; a counter
// that would overflow its field raises ctl->overflow (ACA_ERANGE) instead of wrapping.
//
// In-place updates (no ping-pong): every word a CTA observes for a neighbour is a value that
// neighbour really held, and words only grow. A cell fires only when its word is below every
// observed neighbour word; by the stale-read argument of fig:amcgen and the
// uniqueness argument of fig:a1c1pe the neighbour's state at the firing
// time equals the observed one, so any interleaving of CTAs and threads yields the unique
// trajectory.
#pragma once
#include <stdint.h>

#include "aca_prim.cuh"
#include "nlog_tables.cuh"

namespace aca {

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
};

struct Geo {
    int ndim;
    int nx, ny, nz;          // local extents (the sharded axis is y in 2-D, z in 3-D)
    int NY, NZ;              // global extents of y and z
    int y0, z0;              // global offset of the shard along the sharded axis
    int sharded;             // 0: periodic wrap inside the storage; 1: halo buffers
    int RB, NB, TSH;         // rank bits, counter bits, time shift (= RB + NB + 1)
};

__device__ __host__ __forceinline__ unsigned long long w_time(unsigned long long w, const Geo& g) { return w >> g.TSH; }
__device__ __host__ __forceinline__ unsigned int w_count(unsigned long long w, const Geo& g) {
    return (unsigned int)((w >> 1) & ((1ull << g.NB) - 1ull));
}
__device__ __host__ __forceinline__ unsigned long long w_pack(unsigned long long t, unsigned long long rank,
                                                              unsigned long long n, unsigned long long sb, const Geo& g) {
    return (t << g.TSH) | (rank << (g.NB + 1)) | (n << 1) | sb;
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
    int law;                             // P3L asynchrony law (0 Poisson, 1 uniform, 2 r^(1/8))
    int rounds;                          // R_max
    int round_mode;                      // 0: CTA barrier per round; 1: no barrier, R rounds; 2: per-warp exit
    int do_hash;
    int early;                           // a10: queue early-rejection candidates
    int bulk;                            // max arrivals committed per cell per fire step (1 = one)
    int defer_tail;                      // tile_rounds: defer a partial last fire chunk to the next round
    int tiles_x, tiles_y, tiles_z;
    int phase;                           // -1: every tile; 0 / 1: tiles of that checkerboard colour
    int row_par0;                        // parity of the shard's first tile row (global colouring)
    unsigned long long thr[14];          // P4 table
    unsigned long long thm[98];          // a10 table, see commit_loop (2 (Z+1)^2 entries)
    FrameParams fr;                      // output frames (off unless aca_run_frames)
    int fast;                            // fire_fast applies (law 0, lambda 1, no ties, no frames, N < 2^32)
    int life;                            // rule 2: asynchronous Game of Life (Moore neighbourhood, P10)
};

__device__ __forceinline__ int wrapi(int v, int n) {
    v %= n;
    return v < 0 ? v + n : v;
}
// v in [-n, 2n): one conditional add/sub instead of an integer division
__device__ __forceinline__ int wrap1(int v, int n) { return v < 0 ? v + n : (v >= n ? v - n : v); }

template <bool ONE>
__device__ __forceinline__ unsigned long long ld_word_t(const KParams& P, int gx, int gy, int gz) {
    const Geo& g = P.g;
    const int x = ONE ? wrap1(gx, g.nx) : wrapi(gx, g.nx);
    if (g.ndim == 2) {
        if (!g.sharded) return P.words[(size_t)(ONE ? wrap1(gy, g.ny) : wrapi(gy, g.ny)) * g.nx + x];
        if (gy < 0) return P.halo_lo[x];
        if (gy >= g.ny) return P.halo_hi[x];
        return P.words[(size_t)gy * g.nx + x];
    }
    const int y = ONE ? wrap1(gy, g.ny) : wrapi(gy, g.ny);
    if (!g.sharded) return P.words[((size_t)(ONE ? wrap1(gz, g.nz) : wrapi(gz, g.nz)) * g.ny + y) * g.nx + x];
    if (gz < 0) return P.halo_lo[(size_t)y * g.nx + x];
    if (gz >= g.nz) return P.halo_hi[(size_t)y * g.nx + x];
    return P.words[((size_t)gz * g.ny + y) * g.nx + x];
}
// Address of the word at (gx, gy, gz) with the same wrap / halo rules (the start of a halo row
// for the face TMA copies).
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
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}"
                 ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
#ifndef MBAR_SUSPEND_NS
#define MBAR_SUSPEND_NS 20000   // try_wait suspend-time hint: waiting warps sleep instead of spinning
#endif
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n\t}"
        ::"r"(smem_u32(bar)), "r"(parity), "r"(MBAR_SUSPEND_NS) : "memory");
}
// global -> shared bulk copy (size % 16 == 0, both addresses 16-B aligned), completes on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// order earlier generic-proxy accesses of shared memory before later async-proxy (TMA) ones
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

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

__device__ __forceinline__ FireOut fire(unsigned long long w, uint32_t ones, int z, unsigned long long c,
                                        const Geo& g, const unsigned long long* thr, const unsigned long long* lr,
                                        const uint32_t* rk, unsigned long long inv_lambda, int tie_bits,
                                        int do_hash, Ctl* ctl, int law = 0, const FrameParams* fr = nullptr) {
    FireOut o;
    const uint32_t k = w_count(w, g);
    if (k == (uint32_t)((1ull << g.NB) - 1ull)) {
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
    const unsigned long long d = delta_q32(r.y, r.z, lr, ACA_LN2_Q48, inv_lambda, tie_bits, law);
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
                                              unsigned long long hash, unsigned int rounds, int phase = -1) {
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
        __threadfence();
        ctl->ticket = 0u;
    }
}

__device__ __forceinline__ unsigned long long cell_id(const Geo& g, int gx, int gy, int gz) {
    return g.ndim == 2 ? (unsigned long long)(gy + g.y0) * g.nx + gx
                       : ((unsigned long long)(gz + g.z0) * g.NY + gy) * g.nx + gx;
}

// Global row-major id of the cell at shard-local coordinates (gx, gy) of a 2-D shard, wrapped
// periodically (the explicit (t, c) tie-break of the Moore neighbourhood, where the packed
// rank cannot order diagonal neighbours across the periodic boundary).
__device__ __forceinline__ long long id2(const Geo& g, int gx, int gy) {
    const int x = wrapi(gx, g.nx), y = wrapi(gy + g.y0, g.NY);
    return (long long)y * g.nx + x;
}

// 32-bit cell id (N < 2^32; the Philox counter word c_hi is then 0)
__device__ __forceinline__ uint32_t cell_id32(const Geo& g, int gx, int gy, int gz) {
    return g.ndim == 2 ? (uint32_t)(gy + g.y0) * (uint32_t)g.nx + (uint32_t)gx
                       : ((uint32_t)(gz + g.z0) * (uint32_t)g.NY + (uint32_t)gy) * (uint32_t)g.nx + (uint32_t)gx;
}
template <int NDIM>
__device__ __forceinline__ uint32_t cell_id32t(const Geo& g, int gx, int gy, int gz) {
    return NDIM == 2 ? (uint32_t)(gy + g.y0) * (uint32_t)g.nx + (uint32_t)gx
                     : ((uint32_t)(gz + g.z0) * (uint32_t)g.NY + (uint32_t)gy) * (uint32_t)g.nx + (uint32_t)gx;
}

// fire() for the common configuration (Poisson law, lambda = 1, tie_bits = 0, no output frames,
// N < 2^32): the same integers with the general branches compiled out. The caller raises the
// overflow flag when ok = false.
__device__ __forceinline__ FireOut fire_fast(unsigned long long w, uint32_t ones, int z, uint32_t c, const Geo& g,
                                             const unsigned long long* thr, const unsigned long long* lr,
                                             const uint32_t* rk, int do_hash) {
    FireOut o;
    const uint32_t k = w_count(w, g);
    o.ok = k != (uint32_t)((1ull << g.NB) - 1ull);
    const uint32_t sb = (uint32_t)(w & 1ull);
    const uint32_t idx = ones + (uint32_t)(z + 1) * sb;
    const u32x4 r = philox4x32_10_rk(k, c, 0u, 0u, rk);
    const uint32_t flip = z == 8 ? ((ones == 3u || (sb && ones == 2u)) ? 1u : 0u) ^ sb
                                 : ((unsigned long long)r.x < thr[idx] ? 1u : 0u);
    uint64_t d = nlog_q32(((uint64_t)r.y << 32) | r.z, lr, ACA_LN2_Q48);
    d = d < 1ull ? 1ull : d;
    o.wnew = (w + (d << g.TSH) + 2ull) ^ (unsigned long long)flip;
    o.flip = flip;
    o.h = 0;
    if (do_hash) o.h = ev_hash(r.w, w >> g.TSH, (unsigned long long)(sb ^ flip));
    return o;
}

// The high-half test of two horizontally adjacent cells (PAIRMAP): cell k (k = 0, 1) is active
// iff ah_k < wh and a candidate iff also ah_k <= m_k (bit `bit0 << k` of em); any equality
// (ah_k == m_k or ah_k == wh) clears `tie`, sending the lane to the exact full-word pass.
// Written with explicit predicates so each decision is one compare and one predicated op.
// The same for one cell (COLMAP).
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

// ------------------------------------------------------------------------ uncompacted tile kernel
// One CTA per tile; the tile plus a one-cell halo (faces only) is staged in shared memory;
// up to R rounds of the local-minimum test. SYNC = false: asynchronous in-place updates
// (fig:a1c1pe semantics inside the tile); SYNC = true: the two barriers of
// fig:s1c1pe, private new words then commit — the exact synchronous round
// whose firing fraction N0/N is the paper's efficiency.
template <int NDIM, int TX, int TY, int TZ, int NT, bool SYNC>
__global__ void __launch_bounds__(NT) tile_kernel(const KParams P) {
    constexpr int SX = TX + 2, SY = TY + 2, SZ = (NDIM == 3) ? TZ + 2 : 1;
    constexpr int NSLOT = SX * SY * SZ;
    constexpr int NCELL = TX * TY * TZ;
    constexpr int CPT = NCELL / NT;
    static_assert(NCELL % NT == 0, "tile must be a multiple of the block");
    constexpr int Z = 2 * NDIM;
    constexpr int SXY = SX * SY;

    if (*(volatile unsigned int*)&P.ctl->done) return;

    extern __shared__ __align__(16) unsigned long long smem[];
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
    volatile unsigned long long* VS = S;   // words may change under us (other threads)

    unsigned long long fired = 0, flips = 0, tested = 0, hacc = 0;
    unsigned int rounds = 0;
    for (int r = 0; r < P.rounds; ++r) {
        int any = 0;
        unsigned long long pend[SYNC ? CPT : 1];
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
            const unsigned long long a = VS[s - 1], b = VS[s + 1], c2 = VS[s - SX], d2 = VS[s + SX];
            bool ok = w < a && w < b && w < c2 && w < d2;
            uint32_t ones = (uint32_t)(a & 1ull) + (uint32_t)(b & 1ull) + (uint32_t)(c2 & 1ull) + (uint32_t)(d2 & 1ull);
            if (NDIM == 3) {
                const unsigned long long e = VS[s - SXY], f = VS[s + SXY];
                ok = ok && w < e && w < f;
                ones += (uint32_t)(e & 1ull) + (uint32_t)(f & 1ull);
            }
            if (!ok) continue;
            const FireOut o = fire(w, ones, Z, cell_id(g, x0 + lx, y0 + ly, z0 + lz), g, thr, lr, P.rk,
                                   P.inv_lambda, P.tie_bits, P.do_hash, P.ctl, P.law, &P.fr);
            if (!o.ok) continue;
            hacc += o.h;
            flips += o.flip;
            ++fired;
            changed |= 1u << k;
            any = 1;
            if (SYNC) {
                pend[SYNC ? k : 0] = o.wnew;
                pmask |= 1u << k;
            } else {
                wreg[k] = o.wnew;
                VS[s] = o.wnew;
            }
        }
        if (SYNC) {
            __syncthreads();                                   // barrier 1 of fig:s1c1pe
#pragma unroll
            for (int k = 0; k < CPT; ++k) {
                if ((pmask >> k) & 1u) {
                    const int i = tid + k * NT;
                    const int lx = i % TX, ly = (i / TX) % TY, lz = i / (TX * TY);
                    const int s = (lz + (NDIM == 3)) * SXY + (ly + 1) * SX + lx + 1;
                    wreg[k] = pend[SYNC ? k : 0];
                    VS[s] = wreg[k];
                }
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
        if ((changed >> k) & 1u) P.words[gi] = wreg[k];
        active += wreg[k] < wlim;
    }
    const unsigned long long s_act = block_sum<NT>(active, red);
    const unsigned long long s_fir = block_sum<NT>(fired, red);
    const unsigned long long s_flp = block_sum<NT>(flips, red);
    const unsigned long long s_tst = block_sum<NT>(tested, red);
    const unsigned long long s_hsh = block_sum<NT>(hacc, red);
    if (tid == 0) finish_launch(P.ctl, s_act, s_fir, s_flp, s_tst, s_hsh, rounds);
}

// Shared-memory layout of tile_tma_kernel (host and device): words (NB_ buffers), the P4/a10
// tables, reduction scratch, 2 mbarriers, then the fire queue(s) (the P3 table is read from
// global memory through L1): per-warp queues of
// CPW/2 + 16 entries (the eligible cells of a warp form an independent set: at most one per
// two cells of each row segment), CPW with a10 candidates, or the work-list's two CTA queues
// plus claim bitmaps and counters.
__host__ __device__ constexpr size_t tma_words(int ndim, int tx, int ty, int tz, int hw = 1) {
    return (((size_t)(tx + 4) * (ty + 2 * hw) * (ndim == 3 ? tz + 2 * hw : 1) + 15) & ~(size_t)15);
}
// per-warp queue of tile_rounds: CPW/2 + 16 own cells (+ 64 redundant ring cells with hw = 2)
__host__ __device__ constexpr int tile_queue_per_warp(int cpw, bool early, int hw) {
    return early ? cpw : cpw / 2 + 16 + (hw == 2 ? 64 : 0);
}
__host__ __device__ constexpr size_t tma_queue_entries(int ncell, int nt, bool wl, bool early, int hw = 1) {
    return wl ? (size_t)ncell + 64 : (size_t)(nt / 32) * tile_queue_per_warp(ncell / (nt / 32), early, hw);
}
__host__ __device__ constexpr size_t tma_smem_bytes(int ndim, int tx, int ty, int tz, int nt, int nbuf, bool wl,
                                                    bool early, int hw = 1) {
    return (tma_words(ndim, tx, ty, tz, hw) * nbuf + 16 + 112 + 512 + nt / 32 + 2) * 8 +
           ((tma_queue_entries(tx * ty * tz, nt, wl, early, hw) * 2 + 15) & ~(size_t)15) +
           (wl ? (size_t)tx * ty * tz / 32 * 8 + 16 : 0);
}

// ------------------------------------------------------------ persistent TMA tile kernel
// The production kernel. Persistent CTAs walk the tiles (the sweep direction alternates
// between launches, so the in-place updates of tiles processed earlier in a launch propagate
// both ways: Gauss-Seidel across tiles). Staging of a full tile: its own rows arrive by TMA
// bulk copies (cp.async.bulk; no other CTA writes these rows), the face halo — words other
// CTAs may be updating — by ordinary 8-byte loads (single-copy atomic). DB: the next tile's
// rows stream into a second buffer while the current tile is processed. Per round each warp
// (i) tests its cells: a 32-bit compare of the high halves (full 64-bit compare only on a
// tie), (ii) compacts the eligible cells with a warp scan, (iii) fires them with all lanes
// busy. A queued cell's neighbourhood is frozen until it fires (no neighbour can pass its
// own test while the cell's lower word is unchanged), so compaction preserves exactness.
// Per-lane counters of one tile visit (32-bit: at most NCELL x R x bulk per visit); the tile
// kernels fold them into 64-bit totals after every visit (TileTotals).
struct TileStats {
    unsigned int fired = 0, flips = 0, tested = 0;
    unsigned long long hacc = 0;
};
struct TileTotals {
    unsigned long long fired = 0, flips = 0, tested = 0;
    __device__ __forceinline__ void fold(TileStats& st) {
        fired += st.fired; flips += st.flips; tested += st.tested;
        st.fired = st.flips = st.tested = 0;
    }
};

// Commit the pending arrivals of the cell in slot s for as long as that is exact (a10):
//  * u = 0 (the cell is below every neighbour): an ordinary arrival, flip iff w0 < thr;
//  * u > 0 neighbours may still change before the arrival: commit it only when the draw
//    rejects the flip for EVERY value of those u spins (w0 >= thm = max threshold over the
//    possible neighbour sums) — "rejected in every consistent world". The arrival then
//    advances t and n and leaves s unchanged, which is what it does in the true trajectory
//    whatever the u neighbours do; the other neighbours' spins are known (they cannot move
//    before the arrival, fig:amcgen stale-read argument PAPER.md:833-871). This is the exact
//    use of the BKL observation that most attempts are rejections.
// thm[(s*(Z+1) + u)*(Z+1) + k] (k = known +1 neighbours) > 2^32 means "wait".
template <int NDIM, int SX, int SXY, bool FASTP = false>
__device__ __forceinline__ void commit_loop(const KParams& P, volatile unsigned long long* VS, int s,
                                            unsigned long long cid, const unsigned long long* thr,
                                            const unsigned long long* thm, const unsigned long long* lr,
                                            unsigned long long wlim, TileStats& st) {
    constexpr int Z = 2 * NDIM;
    const Geo& g = P.g;
    unsigned long long w = VS[s];
    for (int it = 0; it < P.bulk; ++it) {
        if (w >= wlim) break;
        const int off[6] = {-1, 1, -SX, SX, -SXY, SXY};
        uint32_t u = 0, k = 0;
#pragma unroll
        for (int q = 0; q < Z; ++q) {
            const unsigned long long nb = VS[s + off[q]];
            const bool below = nb < w;
            u += below;
            k += below ? 0u : (uint32_t)(nb & 1ull);
        }
        const uint32_t sb = (uint32_t)(w & 1ull);
        const unsigned long long tm = thm[(sb * (Z + 1) + u) * (Z + 1) + k];
        if (tm > (1ull << 32)) break;                     // must wait for the u neighbours
        const uint32_t n = w_count(w, g);
        if (n == (uint32_t)((1ull << g.NB) - 1ull)) { atomicOr(&P.ctl->overflow, 1u); break; }
        // FASTP (P.fast: Poisson, lambda = 1, no tie stress, no frames, N < 2^32): the same
        // integers with the general branches compiled out
        const u32x4 r = philox4x32_10_rk(n, (uint32_t)cid, FASTP ? 0u : (uint32_t)(cid >> 32), 0u, P.rk);
        uint32_t flip = 0;
        if (u == 0) flip = (unsigned long long)r.x < thr[k + (uint32_t)(Z + 1) * sb] ? 1u : 0u;
        else if ((unsigned long long)r.x < tm) break;     // a flip is possible in some world: wait
        unsigned long long d;
        if constexpr (FASTP) {
            d = nlog_q32(((uint64_t)r.y << 32) | r.z, lr, ACA_LN2_Q48);
            d = d < 1ull ? 1ull : d;
        } else {
            d = delta_q32(r.y, r.z, lr, ACA_LN2_Q48, P.inv_lambda, P.tie_bits, P.law);
        }
        if (P.do_hash) st.hacc += ev_hash(r.w, w >> g.TSH, (unsigned long long)(sb ^ flip));
        if (!FASTP && P.fr.nb) {
            const unsigned long long tp = w >> g.TSH;
            frame_write(P.fr, tp, tp + d, cid, sb ^ flip);
        }
        w = (w + (d << g.TSH) + 2ull) ^ (unsigned long long)flip;
        VS[s] = w;
        st.flips += flip;
        ++st.fired;
    }
}

// Exact local-minimum test of the cell in slot s against its observed neighbours (P6:
// word order = (t, c) order). High halves first; the full words only on a tie.
template <int NDIM, int SX, int SXY>
__device__ __forceinline__ bool is_local_min(const volatile unsigned long long* VS, const volatile unsigned int* VH,
                                             int s, unsigned long long w) {
    const unsigned int oh = (unsigned int)(w >> 32);
    unsigned int mn = min(min(VH[2 * (s - 1) + 1], VH[2 * (s + 1) + 1]), min(VH[2 * (s - SX) + 1], VH[2 * (s + SX) + 1]));
    if (NDIM == 3) mn = min(mn, min(VH[2 * (s - SXY) + 1], VH[2 * (s + SXY) + 1]));
    if (oh != mn) return oh < mn;
    bool e = w < VS[s - 1] && w < VS[s + 1] && w < VS[s - SX] && w < VS[s + SX];
    if (NDIM == 3) e = e && w < VS[s - SXY] && w < VS[s + SXY];
    return e;
}

// Ring cell ri of a 2-D tile with a 2-wide halo: the (TX+2) x (TY+2) frame around the tile
// (rows -1 and TY over lx = -1..TX, then columns -1 and TX over ly = 0..TY-1).
template <int TX, int TY>
__device__ __forceinline__ void ring_coords(int ri, int& lx, int& ly) {
    if (ri < 2 * (TX + 2)) { ly = ri < TX + 2 ? -1 : TY; lx = ri % (TX + 2) - 1; }
    else { const int r2 = ri - 2 * (TX + 2); lx = r2 < TY ? -1 : TX; ly = r2 % TY; }
}

template <int NDIM, int TX, int TY, int TZ, int NT, bool FULL, bool EARLY, int HW = 1, bool MOORE = false>
__device__ __forceinline__ unsigned int tile_rounds(const KParams& P, unsigned long long* S, unsigned short* Q,
                                                    const unsigned long long* thr, const unsigned long long* thm,
                                                    const unsigned long long* lr, int x0, int y0, int z0,
                                                    unsigned long long wlim, TileStats& st) {
    static_assert(HW == 1 || (HW == 2 && NDIM == 2 && !EARLY), "2-wide halo: 2-D, no a10");
    static_assert(!MOORE || (NDIM == 2 && HW == 1 && !EARLY), "Moore neighbourhood: 2-D V0 only");
    constexpr int SX = TX + 4, SY = TY + 2 * HW;
    constexpr int SXY = SX * SY;
    constexpr int NCELL = TX * TY * TZ;
    constexpr int NW = NT / 32;
    constexpr int CPW = NCELL / NW;
    constexpr int JPL = CPW / 32;
    constexpr int Z = MOORE ? 8 : 2 * NDIM;
    constexpr bool FASTMAP = (TX % 32 == 0) && (CPW % TX == 0) && (TY % (CPW / TX == 0 ? 1 : CPW / TX) == 0);
    constexpr int LPR = TX / 32 > 0 ? TX / 32 : 1;
    const Geo& g = P.g;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wbase = warp * CPW;
    constexpr int QW = tile_queue_per_warp(CPW, EARLY, HW);   // per-warp queue (see tma_smem_bytes)
    unsigned short* q = Q + warp * QW;
    volatile unsigned long long* VS = S;
    const volatile unsigned int* VH = (const volatile unsigned int*)S;   // [2s+1]: high half, [2s]: low half
    auto slot = [](int lx, int ly, int lz) { return (lz + (NDIM == 3 ? HW : 0)) * SXY + (ly + HW) * SX + lx + 2; };
    // 2-wide halo: the inner halo ring (cells of the neighbour tiles) is also advanced here and
    // written back, its arrivals counted here (the owners continue from the new states). A ring
    // cell may fire only if its owner tile is idle during this launch (the other checkerboard
    // colour): then it and its neighbours were last written by finished launches, every state
    // it observes precedes its pending arrival, and the stale-read argument of fig:amcgen
    // applies; it has exactly one writer. Frozen instead: corner cells (diagonal tiles share
    // our colour and run concurrently), the end cells of every edge (corner cells of the neighbour
    // tile, which touch a second active tile), edges whose wrapped neighbour tile has our colour
    // (odd tile counts), rows outside the shard (halo buffers hold one row), ragged tiles, and
    // everything when the launch is not a checkerboard phase. Each thread owns up to two ring
    // cells.
    constexpr int NRING = HW == 2 ? 2 * (TX + 2) + 2 * TY : 0;
    int rs[2] = {0, 0};
    bool rv[2] = {false, false};
    if constexpr (HW == 2) {
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int ri = tid + k * NT;
            if (ri < NRING) {
                int lx, ly;
                ring_coords<TX, TY>(ri, lx, ly);
                rs[k] = slot(lx, ly, 0);
                const int dx = lx < 0 ? -1 : (lx >= TX ? 1 : 0), dy = ly < 0 ? -1 : (ly >= TY ? 1 : 0);
                const int tx = x0 / TX, ty = y0 / TY;
                bool ok = FULL && P.phase >= 0 && (dx == 0 || dy == 0);
                // the two end cells of each edge are corner cells of the neighbour tile, adjacent
                // to a second active tile as well: frozen, so every ring cell has one writer
                if (dy != 0) ok = ok && lx != 0 && lx != TX - 1;
                if (dx != 0) ok = ok && ly != 0 && ly != TY - 1;
                if (dy != 0 && g.sharded) ok = ok && (ty + dy >= 0 && ty + dy < P.tiles_y);
                const int ntx = wrapi(tx + dx, P.tiles_x), nty = wrapi(ty + dy, P.tiles_y);
                ok = ok && (((ntx + nty + P.row_par0) & 1) != ((tx + ty + P.row_par0) & 1));
                rv[k] = ok;
            }
        }
    }
    // PAIRMAP (2-D, 64-wide tiles): lane `lane` owns the column pair (2 lane, 2 lane + 1) of the
    // warp's CPW / TX rows; cell j is row j / 2, column 2 lane + j % 2. The test then reads each
    // row pair with one 128-bit load and reuses every loaded row as the neighbour row of the
    // next: 1.5 loads per cell instead of 5. Otherwise lane `lane` owns columns lane + 32 k.
    constexpr int RPW = CPW / TX;
    constexpr bool PAIRMAP = NDIM == 2 && TX == 64 && HW == 1 && !MOORE && CPW % TX == 0 &&
                             RPW % 2 == 0 && JPL == 2 * RPW;
    // COLMAP (3-D, 32-wide tiles, one z-plane per warp): lane `lane` owns column `lane` of the
    // warp's plane and walks its rows, reusing each row as the y-neighbour of the next (5 loads
    // per cell instead of 7).
    constexpr bool COLMAP = NDIM == 3 && TX == 32 && HW == 1 && !MOORE && !EARLY && CPW == TX * TY && JPL == TY;
    int s0 = 0;
    if (PAIRMAP) {
        s0 = slot(2 * lane, warp * RPW, 0);
    } else if (FASTMAP) {
        const int row0 = warp * (CPW / TX);
        s0 = slot(lane, row0 % TY, row0 / TY);
    }
    unsigned int rounds = 0;
    auto cell_o = [&](int j) {   // tile-local cell index of the lane's j-th cell
        if (PAIRMAP) return wbase + (j >> 1) * TX + 2 * lane + (j & 1);
        return wbase + lane + 32 * j;
    };
    auto cell_slot = [&](int j) {
        if (PAIRMAP) return s0 + (j >> 1) * SX + (j & 1);
        if (FASTMAP) return s0 + (j / LPR) * SX + 32 * (j % LPR);
        const int o = cell_o(j);
        return slot(o % TX, (o / TX) % TY, o / (TX * TY));
    };
    auto cell_valid = [&](int j) {
        if (FULL) return true;
        const int o = cell_o(j);
        const int lx = o % TX, ly = (o / TX) % TY, lz = o / (TX * TY);
        return x0 + lx < g.nx && y0 + ly < g.ny && (NDIM == 2 || z0 + lz < g.nz);
    };
    uint32_t fl32 = 0, fi32 = 0;   // fast-path flips / fires (folded into st at the end)
    // Carried fire chunk (P.defer_tail, 1-cell halo): a round fires whole 32-lane chunks only;
    // its partial last chunk moves to the front of the warp's queue and fires first in the next
    // round (or in the last round, which fires everything). A carried cell stays a local minimum
    // (its neighbours cannot pass it before it fires), so it is exact; its owner lane keeps it
    // in `pend` so it is not queued twice.
    const bool carry_on = HW == 1 && P.defer_tail;
    uint32_t pend = 0;
    int carry = 0;
    for (int r = 0; r < P.rounds; ++r) {
        uint32_t emask = 0, amask = 0;
        int ntest = 0;   // PAIRMAP counts tested cells directly
        if constexpr (!EARLY) {
            // Branch-free test in batches of TB cells: every load of the batch is issued before
            // any compare (the lane's cells are independent), the 32-bit high halves decide
            // unless they tie; tied cells are settled on the full words in a rare second pass.
            constexpr int TB = 4;
            static_assert(JPL % TB == 0, "cells per lane must be a multiple of the test batch");
            uint32_t tmask = 0;
            if constexpr (PAIRMAP) {
                const unsigned int wh = (unsigned int)(wlim >> 32);
                unsigned int tiec = ~0u;
                // rows of the lane's column pair, top to bottom; `a` holds row rr, `b` row rr + 1
                const ulonglong2 up = lds128v(&VS[s0 - SX]);
                unsigned int uh0 = (unsigned int)(up.x >> 32), uh1 = (unsigned int)(up.y >> 32);
                ulonglong2 a = lds128v(&VS[s0]);
#pragma unroll
                for (int rr = 0; rr < RPW; ++rr) {
                    const int sr = s0 + rr * SX;
                    const ulonglong2 b = lds128v(&VS[sr + SX]);   // row rr + 1 (halo row for the last)
                    const unsigned int lh = VH[2 * (sr - 1) + 1], rh = VH[2 * (sr + 2) + 1];
                    const unsigned int ah0 = (unsigned int)(a.x >> 32), ah1 = (unsigned int)(a.y >> 32);
                    const unsigned int m0 = min(min(lh, ah1), min(uh0, (unsigned int)(b.x >> 32)));
                    const unsigned int m1 = min(min(ah0, rh), min(uh1, (unsigned int)(b.y >> 32)));
                    const int j = 2 * rr;
                    // Decided on the 32-bit high halves: active iff high(w) < high(wlim), eligible
                    // iff high(w) <= the neighbours' minimum. A lane that sees any equality (with a
                    // neighbour, or with the T bucket) redoes its cells on the full words below.
                    if constexpr (FULL) {
                        pair_test(ah0, ah1, m0, m1, wh, 1u << j, emask, ntest, tiec);
                    } else {
                        if (cell_valid(j) && ah0 < wh) {
                            ++ntest;
                            if (ah0 <= m0) emask |= 1u << j;
                        }
                        if (cell_valid(j + 1) && ah1 < wh) {
                            ++ntest;
                            if (ah1 <= m1) emask |= 2u << j;
                        }
                        if (ah0 == m0 || ah0 == wh || ah1 == m1 || ah1 == wh) tiec = 0u;
                    }
                    uh0 = ah0; uh1 = ah1;
                    a = b;
                }
                if (tiec == 0u) {   // rare: exact test of the lane's cells on the full words
                    emask = 0;
                    ntest = 0;
#pragma unroll 1
                    for (int j = 0; j < JPL; ++j) {
                        const int sj = cell_slot(j);
                        const unsigned long long w = VS[sj];
                        if (!cell_valid(j) || w >= wlim) continue;
                        ++ntest;
                        if (w < VS[sj - 1] && w < VS[sj + 1] && w < VS[sj - SX] && w < VS[sj + SX]) emask |= 1u << j;
                    }
                }
            } else if constexpr (COLMAP) {
                const unsigned int wh = (unsigned int)(wlim >> 32);
                unsigned int tiec = ~0u;
                unsigned int uh = VH[2 * (s0 - SX) + 1];
                unsigned long long a = VS[s0];
#pragma unroll
                for (int rr = 0; rr < TY; ++rr) {
                    const int sr = s0 + rr * SX;
                    const unsigned long long b = VS[sr + SX];   // row rr + 1 (halo row for the last)
                    const unsigned int ah = (unsigned int)(a >> 32);
                    const unsigned int m = min(min(min(VH[2 * (sr - 1) + 1], VH[2 * (sr + 1) + 1]),
                                                   min(VH[2 * (sr - SXY) + 1], VH[2 * (sr + SXY) + 1])),
                                               min(uh, (unsigned int)(b >> 32)));
                    if constexpr (FULL) {
                        one_test(ah, m, wh, 1u << rr, emask, ntest, tiec);
                    } else {
                        if (cell_valid(rr) && ah < wh) {
                            ++ntest;
                            if (ah <= m) emask |= 1u << rr;
                        }
                        if (ah == m || ah == wh) tiec = 0u;
                    }
                    uh = ah;
                    a = b;
                }
                if (tiec == 0u) {   // rare: exact test of the lane's cells on the full words
                    emask = 0;
                    ntest = 0;
#pragma unroll 1
                    for (int j = 0; j < JPL; ++j) {
                        const int sj = cell_slot(j);
                        const unsigned long long w = VS[sj];
                        if (!cell_valid(j) || w >= wlim) continue;
                        ++ntest;
                        if (w < VS[sj - 1] && w < VS[sj + 1] && w < VS[sj - SX] && w < VS[sj + SX] &&
                            w < VS[sj - SXY] && w < VS[sj + SXY])
                            emask |= 1u << j;
                    }
                }
            } else
#pragma unroll
            for (int j0 = 0; j0 < JPL; j0 += TB) {
                unsigned long long wv[TB];
                unsigned int mv[TB];
#pragma unroll
                for (int k = 0; k < TB; ++k) wv[k] = VS[cell_slot(j0 + k)];
#pragma unroll
                for (int k = 0; k < TB; ++k) {
                    const int s = cell_slot(j0 + k);
                    unsigned int m = min(min(VH[2 * (s - 1) + 1], VH[2 * (s + 1) + 1]),
                                         min(VH[2 * (s - SX) + 1], VH[2 * (s + SX) + 1]));
                    if (NDIM == 3) m = min(m, min(VH[2 * (s - SXY) + 1], VH[2 * (s + SXY) + 1]));
                    if (MOORE)
                        m = min(min(m, min(VH[2 * (s - SX - 1) + 1], VH[2 * (s - SX + 1) + 1])),
                                min(VH[2 * (s + SX - 1) + 1], VH[2 * (s + SX + 1) + 1]));
                    mv[k] = m;
                }
#pragma unroll
                for (int k = 0; k < TB; ++k) {
                    const bool act = cell_valid(j0 + k) && wv[k] < wlim;
                    const unsigned int oh = (unsigned int)(wv[k] >> 32);
                    emask |= (uint32_t)(act && oh < mv[k]) << (j0 + k);
                    tmask |= (uint32_t)(act && oh == mv[k]) << (j0 + k);
                    amask |= (uint32_t)act << (j0 + k);
                }
            }
            while (tmask) {   // tie in the high halves: decide on the full words
                const int j = __ffs(tmask) - 1;
                tmask &= tmask - 1u;
                const int s = cell_slot(j);
                const unsigned long long w = VS[s];
                bool e;
                if (MOORE) {   // rank bits are 0: compare the times, then the cell ids
                    const int o = cell_o(j);
                    const int lx = o % TX, ly = (o / TX) % TY;
                    const unsigned long long t = w >> g.TSH;
                    const long long cs = id2(g, x0 + lx, y0 + ly);
                    e = true;
#pragma unroll
                    for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
                        for (int dx = -1; dx <= 1; ++dx) {
                            if (dx == 0 && dy == 0) continue;
                            const unsigned long long tn = VS[s + dy * SX + dx] >> g.TSH;
                            e = e && (t < tn || (t == tn && cs < id2(g, x0 + lx + dx, y0 + ly + dy)));
                        }
                } else {
                    e = w < VS[s - 1] && w < VS[s + 1] && w < VS[s - SX] && w < VS[s + SX];
                    if (NDIM == 3) e = e && w < VS[s - SXY] && w < VS[s + SXY];
                }
                emask |= (uint32_t)e << j;
            }
            if constexpr (HW == 2) {   // the lane's ring cells take mask bits JPL, JPL + 1
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    if (!rv[k]) continue;
                    const unsigned long long w = VS[rs[k]];
                    const bool act = w < wlim;
                    if (act && is_local_min<NDIM, SX, SXY>(VS, VH, rs[k], w)) emask |= 1u << (JPL + k);
                }
            }
        } else if constexpr (PAIRMAP) {
            // a10 with the column-pair walk: the four neighbours' full words are in registers,
            // so u (neighbours below) and k (+1 spins among the others) come from one pass;
            // u = 0 is the local minimum (words are distinct), else the a10 table decides
            const ulonglong2 up = lds128v(&VS[s0 - SX]);
            unsigned long long u0 = up.x, u1 = up.y;
            ulonglong2 a = lds128v(&VS[s0]);
            auto early_cell = [&](unsigned long long w, unsigned long long n0, unsigned long long n1,
                                  unsigned long long n2, unsigned long long n3, int j) {
                if (!cell_valid(j) || w >= wlim) return;
                ++ntest;
                const uint32_t b0 = n0 < w, b1 = n1 < w, b2 = n2 < w, b3 = n3 < w;
                const uint32_t u = b0 + b1 + b2 + b3;
                const uint32_t k = (b0 ? 0u : (uint32_t)(n0 & 1ull)) + (b1 ? 0u : (uint32_t)(n1 & 1ull)) +
                                   (b2 ? 0u : (uint32_t)(n2 & 1ull)) + (b3 ? 0u : (uint32_t)(n3 & 1ull));
                const bool e = u == 0u || thm[((uint32_t)(w & 1ull) * (Z + 1) + u) * (Z + 1) + k] <= (1ull << 32);
                emask |= (uint32_t)e << j;
            };
#pragma unroll
            for (int rr = 0; rr < RPW; ++rr) {
                const int sr = s0 + rr * SX;
                const ulonglong2 b = lds128v(&VS[sr + SX]);
                const unsigned long long lw = VS[sr - 1], rw = VS[sr + 2];
                early_cell(a.x, lw, a.y, u0, b.x, 2 * rr);
                early_cell(a.y, a.x, rw, u1, b.y, 2 * rr + 1);
                u0 = a.x; u1 = a.y;
                a = b;
            }
        } else
#pragma unroll
        for (int j = 0; j < JPL; ++j) {
            int s;
            bool valid = true;
            if (FASTMAP) {
                s = s0 + (j / LPR) * SX + 32 * (j % LPR);
            } else {
                const int o = wbase + lane + 32 * j;
                s = slot(o % TX, (o / TX) % TY, o / (TX * TY));
            }
            if (!FULL) {
                const int o = wbase + lane + 32 * j;
                const int lx = o % TX, ly = (o / TX) % TY, lz = o / (TX * TY);
                valid = x0 + lx < g.nx && y0 + ly < g.ny && (NDIM == 2 || z0 + lz < g.nz);
            }
            const unsigned long long w = VS[s];
            const bool act = valid && w < wlim;
            if (act) {
                const unsigned int oh = (unsigned int)(w >> 32);
                unsigned int mn = min(min(VH[2 * (s - 1) + 1], VH[2 * (s + 1) + 1]),
                                      min(VH[2 * (s - SX) + 1], VH[2 * (s + SX) + 1]));
                if (NDIM == 3) mn = min(mn, min(VH[2 * (s - SXY) + 1], VH[2 * (s + SXY) + 1]));
                bool e = oh < mn;
                if (oh == mn) {   // tie in the high halves: decide on the full words
                    e = w < VS[s - 1] && w < VS[s + 1] && w < VS[s - SX] && w < VS[s + SX];
                    if (NDIM == 3) e = e && w < VS[s - SXY] && w < VS[s + SXY];
                }
                if (EARLY && !e) {   // early-rejection candidate? (a10; decided in commit_loop)
                    uint32_t u = 0, k = 0;
                    const int off[6] = {-1, 1, -SX, SX, -SXY, SXY};
#pragma unroll
                    for (int q2 = 0; q2 < Z; ++q2) {
                        const unsigned long long nb = VS[s + off[q2]];
                        const bool below = nb < w;
                        u += below;
                        k += below ? 0u : (uint32_t)(nb & 1ull);
                    }
                    e = thm[((w & 1ull) * (Z + 1) + u) * (Z + 1) + k] <= (1ull << 32);
                }
                emask |= (uint32_t)e << j;
            }
            amask |= (uint32_t)act << j;
        }
        st.tested += __popc(amask) + ntest;
        emask &= ~pend;   // carried cells are queued already
        const int mine = __popc(emask);
        int incl = mine;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += v;
        }
        const int cnt = carry + __shfl_sync(0xffffffffu, incl, 31);
        int pos = carry + incl - mine;
        const int nfire = (carry_on && r < P.rounds - 1 && cnt > 32) ? (cnt & ~31) : cnt;
        pend = 0;
        if (carry_on) {
            while (emask) {
                const int j = __ffs(emask) - 1;
                emask &= emask - 1u;
                if (pos >= nfire) pend |= 1u << j;
                q[pos++] = (unsigned short)cell_o(j);
            }
        } else if constexpr (PAIRMAP) {
            // entry of cell j = base + (j / 2) TX + j % 2 = base | ((j << 5) & 0x1c0) | (j & 1)
            // (base = warp CPW + 2 lane has no bits in 0x1c1); highest bit first
            static_assert(TX == 64 && RPW <= 8, "PAIRMAP entry packing");
            uint32_t qp = smem_u32(q) + 2u * (uint32_t)pos;
            const uint32_t base = (uint32_t)(wbase + 2 * lane);
            while (emask) {
                uint32_t j;
                asm("bfind.u32 %0, %1;" : "=r"(j) : "r"(emask));
                emask ^= 1u << j;
                const uint32_t e = base | ((j << 5) & 0x1c0u) | (j & 1u);
                asm volatile("st.shared.u16 [%0], %1;" ::"r"(qp), "h"((unsigned short)e) : "memory");
                qp += 2u;
            }
        } else {
            while (emask) {
                const int j = __ffs(emask) - 1;
                emask &= emask - 1u;
                q[pos++] = (unsigned short)((HW == 1 || j < JPL) ? cell_o(j) : NCELL + tid + (j - JPL) * NT);
            }
        }
        __syncwarp();
        if ((PAIRMAP || COLMAP) && !EARLY && P.fast) {
            // The common case (64-wide 2-D / 32-wide 3-D tiles, Poisson, lambda = 1, no frames):
            // the queue and the words are addressed with 32-bit shared-window offsets.
            const uint32_t qa = smem_u32(q), sa = smem_u32(S);
            const uint32_t cb = (uint32_t)(y0 + g.y0) * (uint32_t)g.nx + (uint32_t)x0;
            for (int i = lane; i < nfire; i += 32) {
                uint32_t o;
                asm volatile("ld.shared.u16 %0, [%1];" : "=r"(o) : "r"(qa + 2u * (uint32_t)i) : "memory");
                // o < NCELL: in 2-D the row is o / TX and there is no plane index
                const uint32_t lx = o % TX, ly = NDIM == 3 ? (o / TX) % TY : o / TX,
                               lz = NDIM == 3 ? o / (TX * TY) : 0u;
                const uint32_t a = sa + 8u * (uint32_t)slot((int)lx, (int)ly, (int)lz);
                unsigned long long w;
                uint32_t b0, b1, b2, b3, b4 = 0, b5 = 0;
                asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(w) : "r"(a) : "memory");
                asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(b0) : "r"(a - 8u) : "memory");
                asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(b1) : "r"(a + 8u) : "memory");
                asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(b2) : "r"(a - 8u * SX) : "memory");
                asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(b3) : "r"(a + 8u * SX) : "memory");
                if constexpr (NDIM == 3) {
                    asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(b4) : "r"(a - 8u * SXY) : "memory");
                    asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(b5) : "r"(a + 8u * SXY) : "memory");
                }
                const uint32_t ones = (b0 & 1u) + (b1 & 1u) + (b2 & 1u) + (b3 & 1u) + (b4 & 1u) + (b5 & 1u);
                const uint32_t cid = NDIM == 2 ? cb + ly * (uint32_t)g.nx + lx
                                               : cell_id32t<NDIM>(g, x0 + (int)lx, y0 + (int)ly, z0 + (int)lz);
                const FireOut f = fire_fast(w, ones, Z, cid, g, thr, lr, P.rk, P.do_hash);
                if (!f.ok) { atomicOr(&P.ctl->overflow, 1u); continue; }
                asm volatile("st.volatile.shared.u64 [%0], %1;" ::"r"(a), "l"(f.wnew) : "memory");
                st.hacc += f.h;
                fl32 += f.flip;
                ++fi32;
            }
        } else
        for (int i = lane; i < nfire; i += 32) {
            const int o = q[i];
            if (HW == 2 && o >= NCELL) {   // ring cell of an idle neighbour tile: a real arrival
                int rlx, rly;
                ring_coords<TX, TY>(o - NCELL, rlx, rly);
                const int s = slot(rlx, rly, 0);
                const unsigned long long w = VS[s];
                const uint32_t ones = (VH[2 * (s - 1)] & 1u) + (VH[2 * (s + 1)] & 1u) + (VH[2 * (s - SX)] & 1u) +
                                      (VH[2 * (s + SX)] & 1u);
                const int gy = y0 + rly;
                const uint32_t c = cell_id32(g, wrapi(x0 + rlx, g.nx), g.sharded ? gy : wrapi(gy, g.ny), 0);
                const FireOut f = fire(w, ones, Z, (unsigned long long)c, g, thr, lr, P.rk, P.inv_lambda, P.tie_bits,
                                       P.do_hash, P.ctl, P.law, &P.fr);
                if (!f.ok) continue;
                VS[s] = f.wnew;
                st.hacc += f.h;
                st.flips += f.flip;
                ++st.fired;
                continue;
            }
            const int lx = o % TX, ly = (o / TX) % TY, lz = o / (TX * TY);
            const int s = slot(lx, ly, lz);
            if (EARLY) {
                if (P.fast)
                    commit_loop<NDIM, SX, SXY, true>(P, VS, s, cell_id32t<NDIM>(g, x0 + lx, y0 + ly, z0 + lz), thr, thm,
                                                     lr, wlim, st);
                else
                    commit_loop<NDIM, SX, SXY>(P, VS, s, cell_id(g, x0 + lx, y0 + ly, z0 + lz), thr, thm, lr, wlim, st);
                continue;
            }
            const unsigned long long w = VS[s];
            uint32_t ones = (VH[2 * (s - 1)] & 1u) + (VH[2 * (s + 1)] & 1u) + (VH[2 * (s - SX)] & 1u) +
                            (VH[2 * (s + SX)] & 1u);
            if (NDIM == 3) ones += (VH[2 * (s - SXY)] & 1u) + (VH[2 * (s + SXY)] & 1u);
            if (MOORE)
                ones += (VH[2 * (s - SX - 1)] & 1u) + (VH[2 * (s - SX + 1)] & 1u) + (VH[2 * (s + SX - 1)] & 1u) +
                        (VH[2 * (s + SX + 1)] & 1u);
            if (P.fast) {   // uniform: Poisson law, lambda = 1, no tie stress, no frames, N < 2^32
                const FireOut f = fire_fast(w, ones, Z, cell_id32t<NDIM>(g, x0 + lx, y0 + ly, z0 + lz), g, thr, lr, P.rk,
                                            P.do_hash);
                if (!f.ok) { atomicOr(&P.ctl->overflow, 1u); continue; }
                VS[s] = f.wnew;
                st.hacc += f.h;
                fl32 += f.flip;
                ++fi32;
                continue;
            }
            const FireOut f = fire(w, ones, Z, cell_id(g, x0 + lx, y0 + ly, z0 + lz), g, thr, lr, P.rk,
                                   P.inv_lambda, P.tie_bits, P.do_hash, P.ctl, P.law, &P.fr);
            if (!f.ok) continue;
            VS[s] = f.wnew;
            st.hacc += f.h;
            st.flips += f.flip;
            ++st.fired;
        }
        // Every queued cell's new word must be visible to the whole warp before its next test:
        // a queued cell is still a local minimum until its word is written, and lanes of a warp
        // are not guaranteed to reconverge after the divergent fire loop.
        __syncwarp();
        if (cnt > nfire) {   // move the partial chunk (< 32 entries) to the queue front
            const int nc = cnt - nfire;
            const unsigned short e = lane < nc ? q[nfire + lane] : (unsigned short)0;
            __syncwarp();
            if (lane < nc) q[lane] = e;
            __syncwarp();
        }
        carry = cnt - nfire;
        ++rounds;
        if (P.round_mode == 0) {
            if (__syncthreads_count(cnt > 0) == 0) break;   // CTA-wide stall detection
        } else if (P.round_mode == 2 && cnt == 0) {
            break;                                          // this warp found nothing eligible
        }
    }
    st.flips += fl32;
    st.fired += fi32;
    if constexpr (HW == 2) {
        // The ring cells this tile advanced are written back: their owner tiles are idle in this
        // launch (single writer, words only grow) and will continue from these states, so the
        // global state stays one in which every neighbour's last arrival precedes a cell's
        // pending arrival. Other warps may still be firing ring cells: wait for all of them.
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            if (!rv[k]) continue;
            int lx, ly;
            ring_coords<TX, TY>(tid + k * NT, lx, ly);
            const int gy = y0 + ly;
            const int gyy = g.sharded ? gy : wrapi(gy, g.ny), gxx = wrapi(x0 + lx, g.nx);
            const size_t gi = (size_t)gyy * g.nx + gxx;
            P.words[gi] = VS[rs[k]];
            push_word(P, gxx, gyy, 0, VS[rs[k]]);
        }
    }
    return rounds;
}

// Register-resident rounds (full tiles whose rows split evenly over the warps). Lane `lane`
// of warp `warp` owns RW rows x CPL adjacent columns; their words live in registers. The
// test of a round reads the row neighbours from the lane's own registers, the column
// neighbours by warp shuffles of the 32-bit high halves (halo columns preloaded into the
// edge lanes' registers), and only the rows at a warp edge (and 3-D plane neighbours) from
// shared memory. All tests of a round see one snapshot (no cell fires during the test
// phase): this is exactly the synchronous round of fig:s1c1pe, whose
// eligible cells are pairwise non-neighbours. They are queued per warp and fired by the
// whole CTA (all lanes busy), then each owner reloads the words of its fired cells.
template <int NDIM, int TX, int TY, int TZ, int NT>
struct RegMap {
    static constexpr int NCELL = TX * TY * TZ;
    static constexpr int NW = NT / 32;
    static constexpr int CPW = NCELL / NW;
    static constexpr int CPL = TX / 32;                 // columns per lane
    static constexpr int RW = CPL > 0 ? CPW / TX : 0;   // rows per warp
    static constexpr bool ok = (TX % 32 == 0) && (CPL == 1 || CPL == 2) && (CPW % TX == 0) && RW >= 2 &&
                               (TY % (RW > 0 ? RW : 1) == 0) && RW * CPL <= 32;
};

template <int NDIM, int TX, int TY, int TZ, int NT>
__device__ __forceinline__ unsigned int tile_rounds_reg(const KParams& P, unsigned long long* S, unsigned short* Q,
                                                        unsigned int* wcnt, const unsigned long long* thr,
                                                        const unsigned long long* lr, int x0, int y0, int z0,
                                                        unsigned long long wlim, TileStats& st) {
    using M = RegMap<NDIM, TX, TY, TZ, NT>;
    constexpr int CPL = M::CPL, RW = M::RW, NW = M::NW, CPW = M::CPW;
    constexpr int SX = TX + 4, SY = TY + 2, SXY = SX * SY;
    constexpr int Z = 2 * NDIM;
    const Geo& g = P.g;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int row0 = warp * RW;                       // first (y, z) row of this warp
    const int ly0 = row0 % TY, lz0 = row0 / TY;
    const int s0 = (lz0 + (NDIM == 3)) * SXY + (ly0 + 1) * SX + lane * CPL + 2;
    volatile unsigned long long* VS = S;
    const volatile unsigned int* VH = (const volatile unsigned int*)S;

    unsigned long long w[RW][CPL];
    unsigned int hx[RW];   // frozen halo column: lane 0 keeps the left one, lane 31 the right one
#pragma unroll
    for (int j = 0; j < RW; ++j) {
#pragma unroll
        for (int c = 0; c < CPL; ++c) w[j][c] = VS[s0 + j * SX + c];
        hx[j] = VH[2 * (s0 + j * SX + (lane == 0 ? -1 : CPL)) + 1];
    }
    unsigned int rounds = 0;
    for (int r = 0; r < P.rounds; ++r) {
        uint32_t emask = 0, ntest = 0;
        // rows just outside the warp (other warps' rows or the tile halo) and plane neighbours
        unsigned int up_e[CPL], dn_e[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            up_e[c] = VH[2 * (s0 - SX + c) + 1];
            dn_e[c] = VH[2 * (s0 + RW * SX + c) + 1];
        }
#pragma unroll
        for (int j = 0; j < RW; ++j) {
            const unsigned int kl = __shfl_up_sync(0xffffffffu, (unsigned int)(w[j][CPL - 1] >> 32), 1);
            const unsigned int kr = __shfl_down_sync(0xffffffffu, (unsigned int)(w[j][0] >> 32), 1);
            const unsigned int left0 = lane > 0 ? kl : hx[j];
            const unsigned int rightN = lane < 31 ? kr : hx[j];
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
                const unsigned long long wc = w[j][c];
                const unsigned int oh = (unsigned int)(wc >> 32);
                const unsigned int kL = c > 0 ? (unsigned int)(w[j][c - 1] >> 32) : left0;
                const unsigned int kR = c < CPL - 1 ? (unsigned int)(w[j][c + 1] >> 32) : rightN;
                const unsigned int kU = j > 0 ? (unsigned int)(w[j - 1][c] >> 32) : up_e[c];
                const unsigned int kD = j < RW - 1 ? (unsigned int)(w[j + 1][c] >> 32) : dn_e[c];
                unsigned int mn = min(min(kL, kR), min(kU, kD));
                const int s = s0 + j * SX + c;
                if (NDIM == 3) mn = min(mn, min(VH[2 * (s - SXY) + 1], VH[2 * (s + SXY) + 1]));
                const bool act = wc < wlim;
                bool e = act && oh < mn;
                if (act && oh == mn) {   // tie in the high halves: full words from shared memory
                    e = wc < VS[s - 1] && wc < VS[s + 1] && wc < VS[s - SX] && wc < VS[s + SX];
                    if (NDIM == 3) e = e && wc < VS[s - SXY] && wc < VS[s + SXY];
                }
                emask |= (uint32_t)e << (j * CPL + c);
                ntest += act;
            }
        }
        st.tested += ntest;
        // compaction into this warp's queue region
        const int mine = __popc(emask);
        int incl = mine;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += v;
        }
        int pos = warp * CPW + incl - mine;
        uint32_t em = emask;
        while (em) {
            const int b = __ffs(em) - 1;
            em &= em - 1u;
            const int j = b / CPL, c = b % CPL;
            const int o = (row0 + j) * TX + lane * CPL + c;   // cell index in the tile
            Q[pos++] = (unsigned short)o;
        }
        if (lane == 31) wcnt[warp] = (unsigned int)incl;
        __syncthreads();
        // CTA-wide fire of all queued cells
        unsigned int cw[NW];
        unsigned int total = 0;
#pragma unroll
        for (int v = 0; v < NW; ++v) { cw[v] = wcnt[v]; total += cw[v]; }
        if (total == 0) break;
        for (unsigned int i = tid; i < total; i += NT) {
            unsigned int acc = 0, qi = 0;
#pragma unroll
            for (int u = 0; u < NW; ++u) {   // queue entry i lives in warp u's region
                if (i >= acc) qi = u * CPW + (i - acc);
                acc += cw[u];
            }
            const int o = Q[qi];
            const int lx = o % TX, ly = (o / TX) % TY, lz = o / (TX * TY);
            const int s = (lz + (NDIM == 3)) * SXY + (ly + 1) * SX + lx + 2;
            const unsigned long long wv = VS[s];
            uint32_t ones = (VH[2 * (s - 1)] & 1u) + (VH[2 * (s + 1)] & 1u) + (VH[2 * (s - SX)] & 1u) +
                            (VH[2 * (s + SX)] & 1u);
            if (NDIM == 3) ones += (VH[2 * (s - SXY)] & 1u) + (VH[2 * (s + SXY)] & 1u);
            const FireOut f = fire(wv, ones, Z, cell_id(g, x0 + lx, y0 + ly, z0 + lz), g, thr, lr, P.rk,
                                   P.inv_lambda, P.tie_bits, P.do_hash, P.ctl, P.law, &P.fr);
            if (!f.ok) continue;
            VS[s] = f.wnew;
            st.hacc += f.h;
            st.flips += f.flip;
            ++st.fired;
        }
        ++rounds;
        __syncthreads();
        // owners reload the words of their fired cells
#pragma unroll
        for (int j = 0; j < RW; ++j)
#pragma unroll
            for (int c = 0; c < CPL; ++c)
                if ((emask >> (j * CPL + c)) & 1u) w[j][c] = VS[s0 + j * SX + c];
    }
    return rounds;
}


// Work-list rounds (full tiles). Round 0 tests every cell of the tile against one snapshot
// and queues the local minima; every later round fires the queued cells and re-tests ONLY
// the cells whose neighbourhood just changed — the fired cell and its in-tile neighbours —
// queueing the new local minima for the next round (a claim bitmap keeps each cell once per
// queue). A cell can become eligible only when it or one of its neighbours fires (words only
// grow; the halo is frozen for the launch), so this finds what a full re-scan would find, at
// about Z + 1 tests per arrival instead of one test per cell per round.
// Exactness: every queued cell was a local minimum when it was queued and stays one until it
// fires (its neighbours, being larger, cannot fire first), so a queue is a set of pairwise
// non-adjacent eligible cells — the set of one synchronous round of fig:s1c1pe
// — and each fires against a neighbourhood frozen until its own write
// (stale-read argument of fig:amcgen). The loop runs until the tile's
// frontier reaches the halo's time bound (empty queue) or R_max rounds.
template <int NDIM, int TX, int TY, int TZ, int NT>
__device__ __forceinline__ unsigned int tile_rounds_wl(const KParams& P, unsigned long long* S, unsigned short* Q,
                                                       unsigned int* claim, unsigned int* qcnt,
                                                       const unsigned long long* thr, const unsigned long long* lr,
                                                       int x0, int y0, int z0, unsigned long long wlim, TileStats& st) {
    constexpr int SX = TX + 4, SY = TY + 2, SXY = SX * SY;
    constexpr int NCELL = TX * TY * TZ;
    constexpr int NW = NT / 32;
    constexpr int CPW = NCELL / NW;
    constexpr int JPL = CPW / 32;
    constexpr int Z = 2 * NDIM;
    constexpr int QH = NCELL / 2 + 32;          // capacity of one queue (an independent set)
    constexpr int NCW = NCELL / 32;             // words of one claim bitmap
    static_assert(CPW % 32 == 0, "whole warps of cells");
    const Geo& g = P.g;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    volatile unsigned long long* VS = S;
    const volatile unsigned int* VH = (const volatile unsigned int*)S;
    volatile unsigned int* VC = qcnt;
    auto slot_of = [](int o) {   // tile cell index -> smem slot
        const int lx = o % TX, ly = (o / TX) % TY, lz = o / (TX * TY);
        return (lz + (NDIM == 3)) * SXY + (ly + 1) * SX + lx + 2;
    };

    for (int i = tid; i < 2 * NCW; i += NT) claim[i] = 0u;
    if (tid < 4) qcnt[tid] = 0u;
    __syncthreads();

    // ---- round 0: full scan against one snapshot (no cell fires before the barrier)
    {
        const int o0 = warp * CPW + lane;
        uint32_t emask = 0, amask = 0;
#pragma unroll
        for (int j = 0; j < JPL; ++j) {
            const int o = o0 + 32 * j;   // rows of this warp, lane-contiguous columns
            const int s = slot_of(o);
            const unsigned long long w = VS[s];
            const bool act = w < wlim;
            if (act && is_local_min<NDIM, SX, SXY>(VS, VH, s, w)) emask |= 1u << j;
            amask |= (uint32_t)act << j;
        }
        st.tested += __popc(amask);
        const int mine = __popc(emask);
        int incl = mine;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += v;
        }
        unsigned int base = 0;
        if (lane == 31 && incl) base = atomicAdd(&qcnt[0], (unsigned int)incl);
        base = __shfl_sync(0xffffffffu, base, 31);
        int pos = (int)base + incl - mine;
        while (emask) {
            const int j = __ffs(emask) - 1;
            emask &= emask - 1u;
            Q[pos++] = (unsigned short)(o0 + 32 * j);
        }
    }
    __syncthreads();

    // ---- fire rounds
    const int doff[6] = {-1, 1, -TX, TX, -TX * TY, TX * TY};
    const int soff[6] = {-1, 1, -SX, SX, -SXY, SXY};
    unsigned int rounds = 1;
    for (int r = 0; r < P.rounds; ++r) {
        const int n = (int)VC[r % 3];
        if (n == 0) break;
        const int cur = r & 1;
        if (tid == 0) VC[(r + 2) % 3] = 0u;                         // counter of the round after next
        for (int i = tid; i < NCW; i += NT) claim[cur * NCW + i] = 0u;   // bitmap of this round's queue
        const unsigned short* qin = Q + cur * QH;
        unsigned short* qout = Q + (cur ^ 1) * QH;
        unsigned int* cl = claim + (cur ^ 1) * NCW;
        unsigned int* cnt_out = qcnt + (r + 1) % 3;
        for (int b0 = warp * 32; b0 < n; b0 += NT) {
            const int i = b0 + lane;
            uint32_t pm = 0;
            int ofired = 0;
            if (i < n) {
                const int o = qin[i];
                const int lx = o % TX, ly = (o / TX) % TY, lz = o / (TX * TY);
                const int s = slot_of(o);
                const unsigned long long w = VS[s];
                uint32_t ones = (VH[2 * (s - 1)] & 1u) + (VH[2 * (s + 1)] & 1u) + (VH[2 * (s - SX)] & 1u) +
                                (VH[2 * (s + SX)] & 1u);
                if (NDIM == 3) ones += (VH[2 * (s - SXY)] & 1u) + (VH[2 * (s + SXY)] & 1u);
                const FireOut f = fire(w, ones, Z, cell_id(g, x0 + lx, y0 + ly, z0 + lz), g, thr, lr, P.rk,
                                       P.inv_lambda, P.tie_bits, P.do_hash, P.ctl, P.law, &P.fr);
                if (f.ok) {
                    VS[s] = f.wnew;
                    st.hacc += f.h;
                    st.flips += f.flip;
                    ++st.fired;
                    // Re-test the cell itself and its in-tile neighbours (halo cells are frozen).
                    // All loads first (independent, in flight together), then the compares;
                    // the fired cell's new word is one of every neighbour's neighbours.
                    const unsigned long long wn = f.wnew;
                    const unsigned int hn = (unsigned int)(wn >> 32);
                    unsigned long long wq[Z];
                    bool inq[Z];
#pragma unroll
                    for (int q = 0; q < Z; ++q) {
                        const int a = q >> 1;
                        const int coord = a == 0 ? lx : (a == 1 ? ly : lz);
                        const int ext = a == 0 ? TX : (a == 1 ? TY : TZ);
                        inq[q] = (q & 1) ? coord != ext - 1 : coord != 0;
                        wq[q] = VS[s + soff[q]];
                    }
                    unsigned int mq[Z];   // min over the high halves of x_q's other neighbours
#pragma unroll
                    for (int q = 0; q < Z; ++q) {
                        unsigned int m = hn;
                        if (inq[q]) {
#pragma unroll
                            for (int p = 0; p < Z; ++p)
                                if (p != (q ^ 1)) m = min(m, VH[2 * (s + soff[q] + soff[p]) + 1]);
                        }
                        mq[q] = m;
                    }
                    uint32_t em = 0, ntest = 0;
                    {   // the fired cell itself
                        unsigned int m = (unsigned int)(wq[0] >> 32);
#pragma unroll
                        for (int q = 1; q < Z; ++q) m = min(m, (unsigned int)(wq[q] >> 32));
                        if (wn < wlim) {
                            ++ntest;
                            const bool e = hn != m ? hn < m : is_local_min<NDIM, SX, SXY>(VS, VH, s, wn);
                            em |= (uint32_t)e;
                        }
                    }
#pragma unroll
                    for (int q = 0; q < Z; ++q) {
                        if (!inq[q] || wq[q] >= wlim) continue;
                        ++ntest;
                        const unsigned int h = (unsigned int)(wq[q] >> 32);
                        const bool e = h != mq[q] ? h < mq[q] : is_local_min<NDIM, SX, SXY>(VS, VH, s + soff[q], wq[q]);
                        em |= (uint32_t)e << (q + 1);
                    }
                    st.tested += ntest;
                    if (em) {   // rare: about one new local minimum per arrival
#pragma unroll
                        for (int q = 0; q <= Z; ++q) {
                            if (!((em >> q) & 1u)) continue;
                            const int oc = q == 0 ? o : o + doff[q - 1];
                            const unsigned int bit = 1u << (oc & 31);
                            if (atomicOr(&cl[oc >> 5], bit) & bit) continue;   // already queued
                            pm |= 1u << q;
                        }
                    }
                    ofired = o;
                }
            }
            // warp-aggregated push into the next queue
            const int mine = __popc(pm);
            int incl = mine;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += v;
            }
            unsigned int base = 0;
            if (lane == 31 && incl) base = atomicAdd(cnt_out, (unsigned int)incl);
            base = __shfl_sync(0xffffffffu, base, 31);
            int pos = (int)base + incl - mine;
#pragma unroll
            for (int q = 0; q <= Z; ++q)
                if ((pm >> q) & 1u) qout[pos++] = (unsigned short)(q == 0 ? ofired : ofired + doff[q - 1]);
        }
        ++rounds;
        __syncthreads();
    }
    return rounds;
}

template <int NDIM, int TX, int TY, int TZ>
__device__ __forceinline__ void halo_coords(int h, int& lx, int& ly, int& lz) {
    lz = 0;
    if (NDIM == 2) {
        if (h < TX) { lx = h; ly = -1; }
        else if (h < 2 * TX) { lx = h - TX; ly = TY; }
        else if (h < 2 * TX + TY) { lx = -1; ly = h - 2 * TX; }
        else { lx = TX; ly = h - 2 * TX - TY; }
    } else {
        int r = h;
        if (r < 2 * TX * TY) { lz = r < TX * TY ? -1 : TZ; r %= TX * TY; lx = r % TX; ly = r / TX; }
        else if ((r -= 2 * TX * TY) < 2 * TX * TZ) { ly = r < TX * TZ ? -1 : TY; r %= TX * TZ; lx = r % TX; lz = r / TX; }
        else { r -= 2 * TX * TZ; lx = r < TY * TZ ? -1 : TX; r %= TY * TZ; ly = r % TY; lz = r / TY; }
    }
}

template <int NDIM, int TX, int TY, int TZ, int NT, int MINB, bool DB, bool REG, bool EARLY = false, bool WL = false,
          int HW = 1, bool MOORE = false>
__global__ void __launch_bounds__(NT, MINB) tile_tma_kernel(const KParams P) {
    static_assert(HW == 1 || (HW == 2 && NDIM == 2 && !EARLY && !WL && !REG && !DB), "2-wide halo: 2-D V0 only");
    constexpr int SX = TX + 4, SY = TY + 2 * HW, SZ = (NDIM == 3) ? TZ + 2 * HW : 1;
    constexpr int SXY = SX * SY;
    constexpr int NSLOT = SXY * SZ;
    constexpr int NSLOTP = (NSLOT + 15) & ~15;          // keep each buffer 128-B aligned
    constexpr int NB_ = DB ? 2 : 1;
    constexpr int NCELL = TX * TY * TZ;
    constexpr int NROWS = TY * TZ;
    constexpr int NW = NT / 32;
    constexpr int NHALO = (NDIM == 2 ? 2 * (TX + TY) : 2 * (TX * TY + TX * TZ + TY * TZ)) + (MOORE ? 4 : 0);
    static_assert(NCELL % NT == 0 && (NCELL / NW) % 32 == 0 && TX % 4 == 0, "tile/block mismatch");

    if (*(volatile unsigned int*)&P.ctl->done) return;

    extern __shared__ __align__(128) unsigned long long smem[];
    unsigned long long* Sb = smem;                                  // NB_ x NSLOTP words
    unsigned long long* thr = Sb + NB_ * NSLOTP;                    // 16
    unsigned long long* thm = thr + 16;                             // 112 (a10 table)
    unsigned long long* lr = thm + 112;                             // 512 (NLOG-2 table, 4 KB)
    unsigned long long* red = lr + 512;                             // NW
    unsigned long long* bar = red + NW;                             // 2
    unsigned short* Q = (unsigned short*)(bar + 2);                 // fire queue(s), see tma_smem_bytes
    unsigned int* claim = (unsigned int*)(Q + ((tma_queue_entries(NCELL, NT, WL, EARLY || REG, HW) + 7) & ~(size_t)7));
    unsigned int* qcnt = claim + 2 * (NCELL / 32);                  // WL: 4 queue counters

    const Geo& g = P.g;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < 16) thr[tid] = tid < 14 ? P.thr[tid] : 0ull;
    for (int i = tid; i < 112; i += NT) thm[i] = i < 98 ? P.thm[i] : ~0ull;
    for (int i = tid; i < 512; i += NT) lr[i] = P.lr[i];
    if (tid == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); }
    __syncthreads();

    auto slot = [](int lx, int ly, int lz) { return (lz + (NDIM == 3 ? HW : 0)) * SXY + (ly + HW) * SX + lx + 2; };
    const unsigned long long wlim = *(volatile unsigned long long*)&P.ctl->wlim;
    // work items: every tile (phase < 0), or the tiles of one checkerboard colour: item k is
    // column pair j = k % hx of tile row k / hx, tx = 2j + ((row parity + phase) & 1)
    const int hx = (P.tiles_x + 1) >> 1;
    const int ntiles = P.phase < 0 ? P.tiles_x * P.tiles_y * P.tiles_z : hx * P.tiles_y * P.tiles_z;
    const bool vec_ok = (g.nx % 2) == 0;
    const bool reverse = P.phase < 0 && ((*(volatile unsigned long long*)&P.ctl->launches) & 1ull);
    TileStats st;
    TileTotals tot;
    unsigned int active = 0;   // cells of this CTA still below T (< 2^32: N < 2^32)
    unsigned int rounds_max = 0;
    uint32_t ph = 0;   // bit b: parity of bar[b]

    auto origin = [&](int it, int& x0, int& y0, int& z0, bool& fast, bool& full) -> bool {
        int tx, ty, tz;
        if (P.phase < 0) {
            const int tile = reverse ? ntiles - 1 - it : it;
            tx = tile % P.tiles_x; ty = (tile / P.tiles_x) % P.tiles_y; tz = tile / (P.tiles_x * P.tiles_y);
        } else {
            const int row = it / hx;
            ty = row % P.tiles_y; tz = row / P.tiles_y;
            tx = 2 * (it % hx) + ((ty + tz + P.row_par0 + P.phase) & 1);
        }
        x0 = tx * TX; y0 = ty * TY; z0 = tz * TZ;
        full = x0 + TX <= g.nx && y0 + TY <= g.ny && (NDIM == 2 || z0 + TZ <= g.nz);
        fast = full && vec_ok;
        return tx < P.tiles_x;
    };
    // FACE_TMA: the halo rows of the y faces (and the z faces in 3-D) are contiguous in x like
    // the tile's own rows, so they arrive by TMA as well (from the wrapped rows or the shard's
    // halo buffers); only the x-face columns are loaded by threads.
    constexpr bool FACE_TMA = HW == 1 && !MOORE;
    constexpr int NFACE = FACE_TMA ? (NDIM == 2 ? 2 : 2 * TY + 2 * TZ) : 0;
    auto issue = [&](int it, int b) {   // warp 0: TMA of the tile's own rows into buffer b
        int x0, y0, z0; bool fast, full;
        if (!origin(it, x0, y0, z0, fast, full) || !fast) return;
        if (lane == 0) mbar_arrive_expect_tx(&bar[b], (uint32_t)(NROWS + NFACE) * TX * 8u);
        __syncwarp();
        fence_proxy_async();
        unsigned long long* S = Sb + b * NSLOTP;
        for (int row = lane; row < NROWS + NFACE; row += 32) {
            if (row < NROWS) {
                const int ly = row % TY, lz = row / TY;
                const size_t gi = NDIM == 2 ? (size_t)(y0 + ly) * g.nx + x0
                                            : ((size_t)(z0 + lz) * g.ny + (y0 + ly)) * g.nx + x0;
                bulk_g2s(&S[slot(0, ly, lz)], P.words + gi, TX * 8, &bar[b]);
            } else {
                const int k = row - NROWS;
                int ly, lz;
                if (NDIM == 2) { ly = k == 0 ? -1 : TY; lz = 0; }
                else if (k < 2 * TY) { lz = k < TY ? -1 : TZ; ly = k % TY; }      // z faces
                else { const int k2 = k - 2 * TY; ly = k2 < TZ ? -1 : TY; lz = k2 % TZ; }   // y faces
                bulk_g2s(&S[slot(0, ly, lz)], word_ptr_t<true>(P, x0, y0 + ly, z0 + lz), TX * 8, &bar[b]);
            }
        }
    };

    if (DB && warp == 0 && (int)blockIdx.x < ntiles) issue(blockIdx.x, 0);
    int k = 0;
    for (int it = blockIdx.x; it < ntiles; it += gridDim.x, ++k) {
        const int b = DB ? (k & 1) : 0;
        unsigned long long* S = Sb + b * NSLOTP;
        int x0, y0, z0; bool fast, full;
        const bool valid = origin(it, x0, y0, z0, fast, full);
        if (warp == 0) {
            if (DB) { if (it + (int)gridDim.x < ntiles) issue(it + gridDim.x, b ^ 1); }
            else issue(it, 0);
        }
        if (!valid) continue;   // odd tiles_x: the last column pair has one tile
        if (fast) {
            if constexpr (FACE_TMA) {   // x-face columns only: left and right of every own row
                for (int h = tid; h < 2 * NROWS; h += NT) {
                    const int row = h >> 1, lx = (h & 1) ? TX : -1, ly = row % TY, lz = row / TY;
                    S[slot(lx, ly, lz)] = ld_word_t<true>(P, x0 + lx, y0 + ly, z0 + lz);
                }
            } else if constexpr (HW == 1) {
                for (int h = tid; h < NHALO; h += NT) {
                    int lx, ly, lz;
                    if (MOORE && h >= NHALO - 4) {   // the four corner cells (diagonal neighbours)
                        const int q = h - (NHALO - 4);
                        lx = (q & 1) ? TX : -1; ly = (q & 2) ? TY : -1; lz = 0;
                    } else {
                        halo_coords<NDIM, TX, TY, TZ>(h, lx, ly, lz);
                    }
                    S[slot(lx, ly, lz)] = ld_word_t<true>(P, x0 + lx, y0 + ly, z0 + lz);
                }
            } else {   // 2-wide halo: rows -2, -1, TY, TY+1 (full width), then columns -2, -1, TX, TX+1
                constexpr int RW = TX + 4, NH2 = 4 * RW + 4 * TY;
                for (int h = tid; h < NH2; h += NT) {
                    int lx, ly;
                    if (h < 4 * RW) { const int r = h / RW; ly = r < 2 ? r - 2 : TY + r - 2; lx = h % RW - 2; }
                    else { const int h2 = h - 4 * RW, c = h2 / TY; lx = c < 2 ? c - 2 : TX + c - 2; ly = h2 % TY; }
                    S[slot(lx, ly, 0)] = ld_word_t<true>(P, x0 + lx, y0 + ly, 0);
                }
            }
            // one warp waits for the TMA rows (the others block in the barrier below without
            // taking issue slots); the barrier then orders the rows before every thread's reads
            if (warp == 0) mbar_wait(&bar[b], (ph >> b) & 1u);
            ph ^= 1u << b;
        } else {
            for (int i = tid; i < NSLOT; i += NT) {
                const int lx = i % SX - 2, ly = (i / SX) % SY - HW, lz = (NDIM == 3) ? i / SXY - HW : 0;
                if (lx < -HW || lx >= TX + HW) continue;
                const int out = (lx < 0 || lx >= TX) + (ly < 0 || ly >= TY) + ((NDIM == 3) && (lz < 0 || lz >= TZ));
                if (HW == 2 || MOORE || out <= 1) S[i] = ld_word(P, x0 + lx, y0 + ly, z0 + lz);
            }
        }
        __syncthreads();

        unsigned int rounds = 0;
        bool done_reg = false;
        if constexpr (WL) {
            if (full) {
                rounds = tile_rounds_wl<NDIM, TX, TY, TZ, NT>(P, S, Q, claim, qcnt, thr, lr, x0, y0, z0, wlim, st);
                done_reg = true;
            }
        } else if constexpr (REG && RegMap<NDIM, TX, TY, TZ, NT>::ok) {
            if (full) {
                rounds = tile_rounds_reg<NDIM, TX, TY, TZ, NT>(P, S, Q, (unsigned int*)red, thr, lr, x0, y0, z0, wlim, st);
                done_reg = true;
            }
        }
        if (!done_reg) {
            rounds = full ? tile_rounds<NDIM, TX, TY, TZ, NT, true, EARLY, HW, MOORE>(P, S, Q, thr, thm, lr, x0, y0, z0,
                                                                                      wlim, st)
                          : tile_rounds<NDIM, TX, TY, TZ, NT, false, EARLY, HW, MOORE>(P, S, Q, thr, thm, lr, x0, y0, z0,
                                                                                       wlim, st);
        }
        rounds_max = rounds > rounds_max ? rounds : rounds_max;
        tot.fold(st);
        // Per-warp write-back: with the per-warp fire queues a warp's own cells (the tile-linear
        // range [warp CPW, (warp + 1) CPW)) are final once its round loop ends, so each warp
        // stores its rows while the others are still firing; one barrier (below) then guards
        // the buffer against the next staging.
        constexpr bool WARP_WB = HW == 1 && !WL && !REG && !DB;
        constexpr int CPW = NCELL / NW;
        if (WARP_WB && fast) {
            const int wb0 = warp * CPW;
            for (int idx = lane; idx < CPW / 2; idx += 32) {
                const int o = wb0 + 2 * idx;
                const int lx = o % TX, ly = (o / TX) % TY, lz = o / (TX * TY);
                const size_t gi = NDIM == 2 ? (size_t)(y0 + ly) * g.nx + x0 + lx
                                            : ((size_t)(z0 + lz) * g.ny + (y0 + ly)) * g.nx + x0 + lx;
                const ulonglong2 v = lds128v(&S[slot(lx, ly, lz)]);
                *reinterpret_cast<ulonglong2*>(P.words + gi) = v;
                active += (v.x < wlim) + (v.y < wlim);
                if (P.push_lo) {
                    const int a = NDIM == 2 ? y0 + ly : z0 + lz, n = NDIM == 2 ? g.ny : g.nz;
                    if (a == 0 || a == n - 1) {
                        const size_t f = NDIM == 2 ? (size_t)(x0 + lx) : (size_t)(y0 + ly) * g.nx + x0 + lx;
                        *reinterpret_cast<ulonglong2*>((a == 0 ? P.push_lo : P.push_hi) + f) = v;
                        if (a == 0 && n == 1) *reinterpret_cast<ulonglong2*>(P.push_hi + f) = v;
                    }
                }
            }
            __syncthreads();   // the buffer is rewritten by a later staging
            continue;
        }
        __syncthreads();

        if (fast) {
            for (int idx = tid; idx < NROWS * (TX / 2); idx += NT) {
                const int row = idx / (TX / 2), m2 = 2 * (idx % (TX / 2));
                const int ly = row % TY, lz = row / TY;
                const size_t gi = NDIM == 2 ? (size_t)(y0 + ly) * g.nx + x0
                                            : ((size_t)(z0 + lz) * g.ny + (y0 + ly)) * g.nx + x0;
                const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(&S[slot(m2, ly, lz)]);
                *reinterpret_cast<ulonglong2*>(P.words + gi + m2) = v;
                active += (v.x < wlim) + (v.y < wlim);
                if (P.push_lo) {
                    const int a = NDIM == 2 ? y0 + ly : z0 + lz, n = NDIM == 2 ? g.ny : g.nz;
                    if (a == 0 || a == n - 1) {
                        const size_t f = NDIM == 2 ? (size_t)(x0 + m2) : (size_t)(y0 + ly) * g.nx + x0 + m2;
                        *reinterpret_cast<ulonglong2*>((a == 0 ? P.push_lo : P.push_hi) + f) = v;
                        if (a == 0 && n == 1) *reinterpret_cast<ulonglong2*>(P.push_hi + f) = v;
                    }
                }
            }
        } else {
            for (int o = tid; o < NCELL; o += NT) {
                const int lx = o % TX, ly = (o / TX) % TY, lz = o / (TX * TY);
                const int gx = x0 + lx, gy = y0 + ly, gz = z0 + lz;
                if (gx < g.nx && gy < g.ny && (NDIM == 2 || gz < g.nz)) {
                    const size_t gi = NDIM == 2 ? (size_t)gy * g.nx + gx : ((size_t)gz * g.ny + gy) * g.nx + gx;
                    const unsigned long long w = S[slot(lx, ly, lz)];
                    P.words[gi] = w;
                    push_word(P, gx, gy, gz, w);
                    active += w < wlim;
                }
            }
        }
        __syncthreads();   // the buffer is rewritten by a later staging
    }
    const unsigned long long s_act = block_sum<NT>((unsigned long long)active, red);
    tot.fold(st);
    const unsigned long long s_fir = block_sum<NT>(tot.fired, red);
    const unsigned long long s_flp = block_sum<NT>(tot.flips, red);
    const unsigned long long s_tst = block_sum<NT>(tot.tested, red);
    const unsigned long long s_hsh = block_sum<NT>(st.hacc, red);
    if (tid == 0) finish_launch(P.ctl, s_act, s_fir, s_flp, s_tst, s_hsh, rounds_max, P.phase);
}

// ------------------------------------------------------------ barrier-free tile pipeline (2-D)
// Variant "async tiles" (ACA_ASYNC_TILES=1; lattices whose shard is a whole number of 64-wide
// tiles with an even tile count per row): two TMA buffers per CTA; each warp waits only for the
// TMA of its tile (mbarrier), loads the x-halo cells of its own rows, runs its rounds and writes
// its own rows back; the last warp to leave a buffer issues the TMA of the CTA's tile after next
// into it. No CTA barrier inside the tile loop: a warp may already work on the next tile while
// its neighbours finish this one (their rows are only read; a warp's cells are fired by that
// warp alone).
template <int TX, int TY, int NT, int MINB, bool EARLY>
__global__ void __launch_bounds__(NT, MINB) tile_as_kernel(const KParams P) {
    constexpr int NDIM = 2, TZ = 1, HW = 1;
    constexpr int SX = TX + 4, SY = TY + 2, SXY = SX * SY;
    constexpr int NSLOTP = (SXY + 15) & ~15;
    constexpr int NCELL = TX * TY, NW = NT / 32, CPW = NCELL / NW, RPW = CPW / TX;
    static_assert(CPW % TX == 0 && 2 * RPW <= 32, "rows per warp");
    if (*(volatile unsigned int*)&P.ctl->done) return;
    extern __shared__ __align__(128) unsigned long long smem[];
    unsigned long long* Sb = smem;                        // 2 x NSLOTP
    unsigned long long* thr = Sb + 2 * NSLOTP;            // 16
    unsigned long long* thm = thr + 16;                   // 112 (entries 98.. are pad)
    unsigned long long* lr = thm + 112;                   // 512
    unsigned long long* red = lr + 512;                   // NW
    unsigned long long* bar = red + NW;                   // 2 full barriers
    unsigned short* Q = (unsigned short*)(bar + 2);
    unsigned int* cnt = (unsigned int*)(thm + 100);       // 2 buffer-release counters (thm pad)
    const Geo& g = P.g;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < 16) thr[tid] = tid < 14 ? P.thr[tid] : 0ull;
    for (int i = tid; i < 112; i += NT) thm[i] = i < 98 ? P.thm[i] : ~0ull;
    for (int i = tid; i < 512; i += NT) lr[i] = P.lr[i];
    __syncthreads();
    if (tid == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); cnt[0] = 0u; cnt[1] = 0u; }
    __syncthreads();
    auto slot = [](int lx, int ly) { return (ly + 1) * SX + lx + 2; };
    const unsigned long long wlim = *(volatile unsigned long long*)&P.ctl->wlim;
    const int hx = P.tiles_x >> 1;
    const int ntiles = P.phase < 0 ? P.tiles_x * P.tiles_y : hx * P.tiles_y;
    const bool reverse = P.phase < 0 && ((*(volatile unsigned long long*)&P.ctl->launches) & 1ull);
    auto origin = [&](int it, int& x0, int& y0) {
        int tx, ty;
        if (P.phase < 0) {
            const int tile = reverse ? ntiles - 1 - it : it;
            tx = tile % P.tiles_x; ty = tile / P.tiles_x;
        } else {
            ty = it / hx;
            tx = 2 * (it % hx) + ((ty + P.row_par0 + P.phase) & 1);
        }
        x0 = tx * TX; y0 = ty * TY;
    };
    auto issue = [&](int it, int b) {   // one warp: TMA of the tile's rows and y-face halo rows
        int x0, y0;
        origin(it, x0, y0);
        if (lane == 0) mbar_arrive_expect_tx(&bar[b], (uint32_t)(TY + 2) * TX * 8u);
        __syncwarp();
        fence_proxy_async();
        unsigned long long* S = Sb + b * NSLOTP;
        for (int row = lane; row < TY + 2; row += 32) {
            const int ly = row < TY ? row : (row == TY ? -1 : TY);
            bulk_g2s(&S[slot(0, ly)], word_ptr_t<true>(P, x0, y0 + ly, 0), TX * 8, &bar[b]);
        }
    };
    if (warp == 0) {
        if ((int)blockIdx.x < ntiles) issue(blockIdx.x, 0);
        if ((int)(blockIdx.x + gridDim.x) < ntiles) issue(blockIdx.x + gridDim.x, 1);
    }
    TileStats st;
    TileTotals tot;
    unsigned int active = 0, rounds_max = 0;
    int k = 0;
    for (int it = blockIdx.x; it < ntiles; it += gridDim.x, ++k) {
        const int b = k & 1;
        unsigned long long* S = Sb + b * NSLOTP;
        int x0, y0;
        origin(it, x0, y0);
        mbar_wait(&bar[b], (uint32_t)((k >> 1) & 1));
        if (lane < 2 * RPW) {   // the x-halo cells of this warp's rows
            const int row = warp * RPW + (lane >> 1), lx = (lane & 1) ? TX : -1;
            S[slot(lx, row)] = ld_word_t<true>(P, x0 + lx, y0 + row, 0);
        }
        __syncwarp();
        const unsigned int rounds = tile_rounds<NDIM, TX, TY, TZ, NT, true, EARLY, HW, false>(
            P, S, Q, thr, thm, lr, x0, y0, 0, wlim, st);
        rounds_max = rounds > rounds_max ? rounds : rounds_max;
        tot.fold(st);
        for (int idx = lane; idx < CPW / 2; idx += 32) {   // write back this warp's rows
            const int o = warp * CPW + 2 * idx;
            const int lx = o % TX, ly = o / TX;
            const size_t gi = (size_t)(y0 + ly) * g.nx + x0 + lx;
            const ulonglong2 v = lds128v(&S[slot(lx, ly)]);
            *reinterpret_cast<ulonglong2*>(P.words + gi) = v;
            active += (v.x < wlim) + (v.y < wlim);
            if (P.push_lo) {
                const int a = y0 + ly;
                if (a == 0 || a == g.ny - 1) {
                    *reinterpret_cast<ulonglong2*>((a == 0 ? P.push_lo : P.push_hi) + x0 + lx) = v;
                    if (a == 0 && g.ny == 1) *reinterpret_cast<ulonglong2*>(P.push_hi + x0 + lx) = v;
                }
            }
        }
        __syncwarp();
        // release the buffer; the last warp out refills it with the tile after next
        unsigned int ticket = 0;
        if (lane == 0) {
            __threadfence_block();
            ticket = atomicAdd(&cnt[b], 1u);
        }
        ticket = __shfl_sync(0xffffffffu, ticket, 0);
        if (ticket == NW - 1) {
            __threadfence_block();
            if (lane == 0) cnt[b] = 0u;
            if (it + 2 * (int)gridDim.x < ntiles) issue(it + 2 * gridDim.x, b);
        }
    }
    __syncthreads();
    tot.fold(st);
    const unsigned long long s_act = block_sum<NT>((unsigned long long)active, red);
    const unsigned long long s_fir = block_sum<NT>(tot.fired, red);
    const unsigned long long s_flp = block_sum<NT>(tot.flips, red);
    const unsigned long long s_tst = block_sum<NT>(tot.tested, red);
    const unsigned long long s_hsh = block_sum<NT>(st.hacc, red);
    if (tid == 0) finish_launch(P.ctl, s_act, s_fir, s_flp, s_tst, s_hsh, rounds_max, P.phase);
}

// ------------------------------------------------------------ whole-lattice kernel
// One CTA holds the entire (small) lattice in shared memory with true periodic addressing
// and runs rounds until no cell has t < T: the whole run_until in one launch. This is the
// configuration-1 "one cell per PE" arrangement (fig:s1c1pe) with the
// 2^14-PE Connection Machine replaced by one CTA.
template <int NT, bool SYNC>
__global__ void __launch_bounds__(NT) whole_kernel(const KParams P) {
    const Geo& g = P.g;
    if (*(volatile unsigned int*)&P.ctl->done) return;
    extern __shared__ __align__(16) unsigned long long smem[];
    const int N = g.nx * g.ny * g.nz;
    unsigned long long* S = smem;                     // N words
    unsigned long long* lr = S + N;                   // 512
    unsigned long long* thr = lr + 512;               // 16
    unsigned long long* red = thr + 16;               // NT/32
    unsigned long long* pend = red + NT / 32;         // N (SYNC only)
    const int tid = threadIdx.x;
    const int Z = 2 * g.ndim;
    for (int i = tid; i < 512; i += NT) lr[i] = P.lr[i];
    if (tid < 16) thr[tid] = tid < 14 ? P.thr[tid] : 0ull;
    for (int i = tid; i < N; i += NT) {
        S[i] = P.words[i];
        if (SYNC) pend[i] = 0ull;
    }
    __syncthreads();
    const unsigned long long wlim = *(volatile unsigned long long*)&P.ctl->wlim;
    unsigned long long fired = 0, flips = 0, tested = 0, hacc = 0;
    unsigned int rounds = 0;
    volatile unsigned long long* VS = S;
    for (;;) {
        int any = 0;
        for (int i = tid; i < N; i += NT) {
            const unsigned long long w = VS[i];
            if (w >= wlim) continue;
            ++tested;
            const int x = i % g.nx, y = (i / g.nx) % g.ny, z = i / (g.nx * g.ny);
            const int row = i - x, pl = g.nx * g.ny;
            const int xm = row + (x == 0 ? g.nx - 1 : x - 1), xp = row + (x == g.nx - 1 ? 0 : x + 1);
            const int ym = i + ((y == 0 ? g.ny - 1 : y - 1) - y) * g.nx;
            const int yp = i + ((y == g.ny - 1 ? 0 : y + 1) - y) * g.nx;
            const unsigned long long a = VS[xm], b = VS[xp], c2 = VS[ym], d2 = VS[yp];
            bool ok = w < a && w < b && w < c2 && w < d2;
            uint32_t ones = (uint32_t)(a & 1ull) + (uint32_t)(b & 1ull) + (uint32_t)(c2 & 1ull) + (uint32_t)(d2 & 1ull);
            if (P.life) {   // Moore neighbourhood, explicit (t, c) order (rank bits are 0)
                const int xmm = x == 0 ? g.nx - 1 : x - 1, xpp = x == g.nx - 1 ? 0 : x + 1;
                const int ymm = y == 0 ? g.ny - 1 : y - 1, ypp = y == g.ny - 1 ? 0 : y + 1;
                const int nbs[8] = {xm, xp, ym, yp, ymm * g.nx + xmm, ymm * g.nx + xpp, ypp * g.nx + xmm,
                                    ypp * g.nx + xpp};
                const unsigned long long t = w >> g.TSH;
                ok = true;
                ones = 0;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const unsigned long long wn = VS[nbs[q]], tn = wn >> g.TSH;
                    ok = ok && (t < tn || (t == tn && i < nbs[q]));
                    ones += (uint32_t)(wn & 1ull);
                }
            }
            if (g.ndim == 3) {
                const int zm = i + ((z == 0 ? g.nz - 1 : z - 1) - z) * pl;
                const int zp = i + ((z == g.nz - 1 ? 0 : z + 1) - z) * pl;
                const unsigned long long e = VS[zm], f = VS[zp];
                ok = ok && w < e && w < f;
                ones += (uint32_t)(e & 1ull) + (uint32_t)(f & 1ull);
            }
            if (!ok) continue;
            const FireOut o = fire(w, ones, P.life ? 8 : Z, (unsigned long long)i, g, thr, lr, P.rk, P.inv_lambda,
                                   P.tie_bits, P.do_hash, P.ctl, P.law, &P.fr);
            if (!o.ok) continue;
            hacc += o.h;
            flips += o.flip;
            ++fired;
            any = 1;
            if (SYNC) pend[i] = o.wnew;   // private new word (0 never occurs: t >= 1)
            else VS[i] = o.wnew;
        }
        ++rounds;
        if (SYNC) {
            __syncthreads();
            for (int i = tid; i < N; i += NT) {
                const unsigned long long pw = pend[i];
                if (pw != 0ull) { S[i] = pw; pend[i] = 0ull; }
            }
        }
        if (__syncthreads_count(any) == 0) break;
    }
    unsigned long long active = 0;
    for (int i = tid; i < N; i += NT) {
        P.words[i] = S[i];
        active += S[i] < wlim;
    }
    const unsigned long long s_act = block_sum<NT>(active, red);
    const unsigned long long s_fir = block_sum<NT>(fired, red);
    const unsigned long long s_flp = block_sum<NT>(flips, red);
    const unsigned long long s_tst = block_sum<NT>(tested, red);
    const unsigned long long s_hsh = block_sum<NT>(hacc, red);
    if (tid == 0) finish_launch(P.ctl, s_act, s_fir, s_flp, s_tst, s_hsh, rounds);
}

// ------------------------------------------------------------------------ init (P5)
__device__ __forceinline__ void cell_coords(const Geo& g, unsigned long long li, unsigned long long& c,
                                            unsigned long long& rank) {
    const unsigned long long x = li % g.nx;
    if (g.ndim == 2) {
        const unsigned long long y = li / g.nx + g.y0;
        c = y * g.nx + x;
        rank = x + y;
    } else {
        const unsigned long long plane = (unsigned long long)g.nx * g.ny;
        const unsigned long long y = (li / g.nx) % g.ny, z = li / plane + g.z0;
        c = (z * g.NY + y) * g.nx + x;
        rank = x + y + z;
    }
}

struct RoundKeys { uint32_t rk[20]; };   // Philox round keys of the seed (philox_round_keys)

__global__ void init_kernel(unsigned long long* __restrict__ words, Geo g, const unsigned long long* __restrict__ lr_g,
                            const RoundKeys K, unsigned long long thr_init, unsigned long long inv_lambda,
                            int tie_bits, unsigned long long n_local, int law) {
    __shared__ unsigned long long lr[512];
    for (int i = threadIdx.x; i < 512; i += blockDim.x) lr[i] = lr_g[i];
    __syncthreads();
    // work items = row segments of 256 cells (x fastest): coordinates without per-cell division
    constexpr int SEG = 256;
    const int nx = g.nx, ny = g.ny, nz = g.ndim == 3 ? g.nz : 1;
    const int nseg = (nx + SEG - 1) / SEG;
    const long long nitems = (long long)ny * nz * nseg;
    for (long long item = blockIdx.x * (long long)(blockDim.x / 32) + (threadIdx.x >> 5); item < nitems;
         item += (long long)gridDim.x * (blockDim.x / 32)) {
        const int row = (int)(item / nseg), sg = (int)(item % nseg);
        const int y = row % ny, z = row / ny;
        const unsigned long long gy = g.ndim == 2 ? (unsigned long long)(y + g.y0) : (unsigned long long)y;
        const unsigned long long gz = g.ndim == 2 ? 0ull : (unsigned long long)(z + g.z0);
        const unsigned long long cbase = g.ndim == 2 ? gy * nx : (gz * g.NY + gy) * nx;
        const int xend = min(nx, (sg + 1) * SEG);
        for (int x = sg * SEG + (threadIdx.x & 31); x < xend; x += 32) {
            const unsigned long long c = cbase + x, rank = (unsigned long long)x + gy + gz;
            const u32x4 r = philox4x32_10_rk(0u, (uint32_t)c, (uint32_t)(c >> 32), 1u, K.rk);
            const unsigned long long sb = ((unsigned long long)r.x < thr_init) ? 0ull : 1ull;
            const unsigned long long t0 = delta_q32(r.y, r.z, lr, ACA_LN2_Q48, inv_lambda, tie_bits, law);
            words[(size_t)row * nx + x] = w_pack(t0, g.RB ? rank : 0ull, 0ull, sb, g);
        }
    }
    (void)n_local;
}

// Frame pre-fill at the start of a frame chunk: every arrival before the chunk is at most the
// previous frame time, so a cell whose pending arrival t is after tau_k held its current spin
// at tau_k. One thread per 32 cells (one u32 word of every frame; no atomics: the chunk's
// kernels run after this one).
__global__ void frame_prefill_kernel(const unsigned long long* __restrict__ words, Geo g, FrameParams F,
                                     unsigned long long n, unsigned long long base_local) {
    for (unsigned long long wi = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; wi * 32 < n;
         wi += (unsigned long long)gridDim.x * blockDim.x) {
        uint32_t acc[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) acc[k] = 0u;
        for (int j = 0; j < 32; ++j) {
            const unsigned long long i = wi * 32 + j;
            if (i >= n) break;
            const unsigned long long w = words[i];
            if (!(w & 1ull)) continue;
            const unsigned long long t = w_time(w, g);
            unsigned long long tau = F.t0;
#pragma unroll
            for (int k = 0; k < 16; ++k, tau += F.dt)
                if (k < F.nb && tau < t) acc[k] |= 1u << j;
        }
        // this shard's cells start at bit base_local (a multiple of 32 when shards are row-aligned)
        const unsigned long long b = base_local + wi * 32;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            if (k >= F.nb || !acc[k]) continue;
            if ((b & 31) == 0) atomicOr(F.bits + (size_t)k * F.wpf + (b >> 5), acc[k]);
            else {   // unaligned shard start: split over two words
                atomicOr(F.bits + (size_t)k * F.wpf + (b >> 5), acc[k] << (b & 31));
                atomicOr(F.bits + (size_t)k * F.wpf + (b >> 5) + 1, acc[k] >> (32 - (b & 31)));
            }
        }
    }
}

// Build words from host-provided spins / times / counters (any may be null: keep the
// current field). Element i of the launch is shard-local cell base + i.
__global__ void pack_kernel(unsigned long long* __restrict__ words, const int8_t* __restrict__ spins,
                            const unsigned long long* __restrict__ times, const unsigned int* __restrict__ counters,
                            Geo g, unsigned long long n, unsigned long long base) {
    if (spins && !times && !counters) {   // spins only: the (t, rank, n) fields are unchanged
        for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
             i += (unsigned long long)gridDim.x * blockDim.x)
            words[i] = (words[i] & ~1ull) | (spins[i] > 0 ? 1ull : 0ull);
        return;
    }
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        unsigned long long c, rank;
        cell_coords(g, base + i, c, rank);
        const unsigned long long w = words[i];
        const unsigned long long t = times ? times[i] : w_time(w, g);
        const unsigned long long k = counters ? counters[i] : w_count(w, g);
        const unsigned long long sb = spins ? (spins[i] > 0 ? 1ull : 0ull) : (w & 1ull);
        words[i] = w_pack(t, g.RB ? rank : 0ull, k, sb, g);
    }
}

// Change the (t, n) split of the words in place (from layout a to layout b).
__global__ void repack_kernel(unsigned long long* __restrict__ words, Geo a, Geo b, unsigned long long n) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long w = words[i];
        const unsigned long long rank = a.RB ? (w >> (a.NB + 1)) & ((1ull << a.RB) - 1ull) : 0ull;
        words[i] = w_pack(w_time(w, a), rank, w_count(w, a), w & 1ull, b);
    }
}

// Gather sampled cells (handle-wide indices; this shard holds [base, base + n)).
__global__ void gather_kernel(const unsigned long long* __restrict__ words, const int64_t* __restrict__ idx,
                              unsigned long long m, long long base, long long n, unsigned long long* __restrict__ w_out) {
    const unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    if (i >= m) return;
    const long long c = idx[i] - base;
    if (c < 0 || c >= n) return;
    w_out[i] = words[c];
}

// Unpack spins (int8), times (u64) or counters (u32) for the getters.
__global__ void unpack_kernel(const unsigned long long* __restrict__ words, int8_t* __restrict__ spins,
                              unsigned long long* __restrict__ times, unsigned int* __restrict__ counters, Geo g,
                              unsigned long long n) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long w = words[i];
        if (spins) spins[i] = (w & 1ull) ? (int8_t)1 : (int8_t)-1;
        if (times) times[i] = w_time(w, g);
        if (counters) counters[i] = w_count(w, g);
    }
}

// Statistics over the owned cells: B (bonds along +e_a), M, sum n, max n, t_min, t_max, and
// the BKL class histogram |Gamma_k| over the (s, Sigma) classes, the
// index of the P4 table (10 classes in 2-D, 14 in 3-D).
struct StatAcc {
    long long bond, mag;
    unsigned long long arrivals, tmin, tmax, nmax;
    unsigned long long hist[14];
};

// a9 statistics of one shard: B, M, sum n, max n, t range and the (s, Sigma) class histogram.
// Each warp walks whole rows (x fastest) in a grid-stride loop over the shard's rows, so the
// neighbour rows are plain pointers (periodic wrap, or the halo rows of a sharded axis) and
// no per-cell division is needed; the histogram is counted with warp ballots (lane b holds
// bin b) instead of shared-memory atomics.
template <int NT>
__global__ void __launch_bounds__(NT) stats_kernel(const KParams P, StatAcc* out, unsigned long long n_local) {
    const Geo& g = P.g;
    const int lane = threadIdx.x & 31;
    const int nwarps = gridDim.x * (NT / 32);
    const int gw = blockIdx.x * (NT / 32) + (threadIdx.x >> 5);
    const int nx = g.nx, ny = g.ny, nz = g.ndim == 3 ? g.nz : 1;
    const int Z = 2 * g.ndim;
    const size_t plane = (size_t)nx * ny;
    long long bond = 0, mag = 0;
    unsigned long long arr = 0, wmin = ~0ull, wmax = 0;
    unsigned int nmax = 0;
    unsigned int hc[14];
#pragma unroll
    for (int b = 0; b < 14; ++b) hc[b] = 0;
    constexpr int SEG = 256;   // cells of a row per work item (8 per lane)
    const int nseg = (nx + SEG - 1) / SEG;
    const int nitems = ny * nz * nseg;
    for (int item = gw; item < nitems; item += nwarps) {
        const int r = item / nseg, sg = item - r * nseg;
        const int y = r % ny, z = r / ny;
        const unsigned long long* cur = P.words + (size_t)r * nx;
        const unsigned long long *yu, *yd, *zu = nullptr, *zd = nullptr;
        if (g.ndim == 2) {
            yu = y + 1 < ny ? cur + nx : (g.sharded ? P.halo_hi : P.words);
            yd = y > 0 ? cur - nx : (g.sharded ? P.halo_lo : P.words + (size_t)(ny - 1) * nx);
        } else {
            yu = y + 1 < ny ? cur + nx : cur - (size_t)(ny - 1) * nx;
            yd = y > 0 ? cur - nx : cur + (size_t)(ny - 1) * nx;
            zu = z + 1 < nz ? cur + plane : (g.sharded ? P.halo_hi + (size_t)y * nx : P.words + (size_t)y * nx);
            zd = z > 0 ? cur - plane
                       : (g.sharded ? P.halo_lo + (size_t)y * nx : P.words + ((size_t)(nz - 1) * ny + y) * nx);
        }
        // per item: 32-bit partial sums, and the histogram as 14 nibble counters (<= 8 cells)
        int ib = 0, im = 0;
        unsigned int ia = 0;
        unsigned long long nib = 0;
        const int xend = min(nx, (sg + 1) * SEG);
#pragma unroll 4
        for (int x = sg * SEG + lane; x < xend; x += 32) {
            const unsigned long long w = cur[x];
            const int sp = (int)(w & 1ull);
            const int xr = x + 1 < nx ? x + 1 : 0, xl = x > 0 ? x - 1 : nx - 1;
            const int ux = (int)(cur[xr] & 1ull), dx = (int)(cur[xl] & 1ull);
            const int uy = (int)(yu[x] & 1ull), dy = (int)(yd[x] & 1ull);
            int ones = ux + dx + uy + dy;
            int plus = 2 * (ux + uy) - 2;
            if (g.ndim == 3) {
                const int uz = (int)(zu[x] & 1ull), dz = (int)(zd[x] & 1ull);
                ones += uz + dz;
                plus += 2 * uz - 1;
            }
            nib += 1ull << (4 * (ones + (Z + 1) * sp));
            const int sv = 2 * sp - 1;
            ib += sv * plus;
            im += sv;
            const unsigned int k = w_count(w, g);
            ia += k;
            nmax = k > nmax ? k : nmax;
            wmin = w < wmin ? w : wmin;   // the time is monotone in the word
            wmax = w > wmax ? w : wmax;
        }
        bond += ib;
        mag += im;
        arr += ia;
#pragma unroll
        for (int b = 0; b < 14; ++b) hc[b] += (unsigned int)(nib >> (4 * b)) & 15u;
    }
    unsigned long long tmin = wmin == ~0ull ? ~0ull : w_time(wmin, g), tmax = w_time(wmax, g);
    unsigned long long nmx = nmax;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        bond += __shfl_xor_sync(0xffffffffu, bond, o);
        mag += __shfl_xor_sync(0xffffffffu, mag, o);
        arr += __shfl_xor_sync(0xffffffffu, arr, o);
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, tmin, o);
        const unsigned long long b = __shfl_xor_sync(0xffffffffu, tmax, o);
        const unsigned long long c = __shfl_xor_sync(0xffffffffu, nmx, o);
        tmin = a < tmin ? a : tmin;
        tmax = b > tmax ? b : tmax;
        nmx = c > nmx ? c : nmx;
#pragma unroll
        for (int b2 = 0; b2 < 14; ++b2) hc[b2] += __shfl_xor_sync(0xffffffffu, hc[b2], o);
    }
    if (lane == 0) {
        atomicAdd((unsigned long long*)&out->bond, (unsigned long long)bond);
        atomicAdd((unsigned long long*)&out->mag, (unsigned long long)mag);
        atomicAdd(&out->arrivals, arr);
        atomicMin(&out->tmin, tmin);
        atomicMax(&out->tmax, tmax);
        atomicMax(&out->nmax, nmx);
#pragma unroll
        for (int b = 0; b < 14; ++b)
            if (hc[b]) atomicAdd(&out->hist[b], (unsigned long long)hc[b]);
    }
    (void)n_local;
}

}  // namespace aca
