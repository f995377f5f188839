// aca_kernels.cuh — sm_100a kernels of the conservative Poisson-asynchronous Ising path.
//
// State in HBM (one shard = a run of rows (2-D) or planes (3-D) of the lattice):
//   words[c] : u64 packed word  (t << SH) | (rank(c) << 1) | [s(c) = +1]
//   cnt[c]   : u32 event counter n(c)
// rank(c) = x + y (+ z) in global coordinates. For every neighbour pair it orders the two
// cells exactly as their row-major ids do (along an axis the ids grow with the coordinate,
// and the periodic pair (n-1, 0) is ordered the same way by both), so one unsigned 64-bit
// compare `w(c) < w(c')` is the lexicographic (t, c) test of P6, and the spin rides in the
// same word: a (t, s) pair is read and written by one 8-byte access and is never torn.
//
// Correctness of in-place updates (no ping-pong): every word a CTA observes for a
// neighbour is a value that neighbour really held, and each cell's word only grows. A cell
// fires only when its word is below every observed neighbour word; by the stale-read
// argument of fig:amcgen and the uniqueness argument of fig:a1c1pe
// the neighbour's state at the firing time equals the observed one, so
// any interleaving of CTAs (and of threads inside a CTA) yields the unique trajectory.
#pragma once
#include <stdint.h>

#include "aca_prim.cuh"
#include "nlog_tables.cuh"

namespace aca {

struct Ctl {                            // device control block, one per shard
    unsigned long long wlim;            // T_q32 << SH: fire iff word < wlim  (t < T)
    unsigned long long active_accum;    // cells with t < T after this launch (accumulating)
    unsigned long long active_last;     // value of the last completed launch
    unsigned long long fired, flips, tested, hash;
    unsigned long long launches, inner_rounds;
    unsigned int done;                  // set when a launch ends with no active cell
    unsigned int ticket;                // last-CTA detection
    unsigned int rounds_max;            // max in-tile rounds over CTAs of this launch
    unsigned int pad;
};

struct Geo {
    int ndim;
    int nx, ny, nz;          // local extents (the sharded axis is y in 2-D, z in 3-D)
    int NY, NZ;              // global extents of y and z
    int y0, z0;              // global offset of the shard along the sharded axis
    int sharded;             // 0: periodic wrap inside the storage; 1: halo buffers
    int SH;                  // packing shift = rank bits + 1
};

struct KParams {
    Geo g;
    unsigned long long* words;
    unsigned int* cnt;
    const unsigned long long* halo_lo;   // sharded axis: row/plane just below the shard
    const unsigned long long* halo_hi;   // ... and just above
    Ctl* ctl;
    const unsigned long long* lr;        // device copy of ACA_NLOG_LR (512 entries)
    uint32_t key0, key1;
    unsigned long long inv_lambda;
    int tie_bits;
    int rounds;                          // R_max
    int do_hash;
    int tiles_x, tiles_y, tiles_z;
    unsigned long long thr[14];          // P4 table
};

__device__ __forceinline__ int wrapi(int v, int n) {
    v %= n;
    return v < 0 ? v + n : v;
}

__device__ __forceinline__ unsigned long long ld_word(const KParams& P, int gx, int gy, int gz) {
    const Geo& g = P.g;
    const int x = wrapi(gx, g.nx);
    if (g.ndim == 2) {
        if (!g.sharded) return P.words[(size_t)wrapi(gy, g.ny) * g.nx + x];
        if (gy < 0) return P.halo_lo[x];
        if (gy >= g.ny) return P.halo_hi[x];
        return P.words[(size_t)gy * g.nx + x];
    }
    const int y = wrapi(gy, g.ny);
    if (!g.sharded) return P.words[((size_t)wrapi(gz, g.nz) * g.ny + y) * g.nx + x];
    if (gz < 0) return P.halo_lo[(size_t)y * g.nx + x];
    if (gz >= g.nz) return P.halo_hi[(size_t)y * g.nx + x];
    return P.words[((size_t)gz * g.ny + y) * g.nx + x];
}

// v in [-n, 2n): one conditional add/sub instead of an integer division
__device__ __forceinline__ int wrap1(int v, int n) { return v < 0 ? v + n : (v >= n ? v - n : v); }

// ---------------------------------------------------------------- TMA bulk-copy helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}"
                 ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
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
// order earlier generic-proxy accesses of shared memory before later async-proxy (TMA) ones
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Block-wide sum of (u64) into ctl via one atomic per CTA.
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
    return s;   // valid in thread 0
}

// One arrival of a cell (fig:a1c1pe steps 3-4; Appendix).
// `ones` = number of +1 neighbours (with multiplicity), z = coordination number.
struct FireOut { unsigned long long wnew; uint32_t flip; unsigned long long h; };

__device__ __forceinline__ FireOut fire(unsigned long long w, uint32_t ones, int z, uint32_t k,
                                        unsigned long long c, int SH, const unsigned long long* thr,
                                        const unsigned long long* lr, uint32_t key0, uint32_t key1,
                                        unsigned long long inv_lambda, int tie_bits, int do_hash) {
    const uint32_t sb = (uint32_t)(w & 1ull);
    const uint32_t idx = ones + (uint32_t)(z + 1) * sb;          // (Sigma+z)/2 + (z+1)(s+1)/2
    const u32x4 r = philox4x32_10(k, (uint32_t)c, (uint32_t)(c >> 32), 0u, key0, key1);
    const uint32_t flip = (unsigned long long)r.x < thr[idx] ? 1u : 0u;
    const unsigned long long d = delta_q32(r.y, r.z, lr, ACA_LN2_Q48, inv_lambda, tie_bits);
    FireOut o;
    o.wnew = (w + (d << SH)) ^ (unsigned long long)flip;
    o.flip = flip;
    o.h = 0;
    if (do_hash) {
        const unsigned long long t = w >> SH;
        o.h = mix64(t ^ rotl64(c, 20) ^ rotl64((unsigned long long)k, 44) ^ (unsigned long long)(sb ^ flip));
    }
    return o;
}

// Last-CTA bookkeeping of one launch: publish counters, decide termination.
__device__ __forceinline__ void finish_launch(Ctl* ctl, unsigned long long active, unsigned long long fired,
                                              unsigned long long flips, unsigned long long tested,
                                              unsigned long long hash, unsigned int rounds) {
    // thread 0 only
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
        const unsigned long long act = atomicAdd(&ctl->active_accum, 0ull);
        ctl->active_last = act;
        ctl->done = (act == 0ull) ? 1u : 0u;
        ctl->active_accum = 0ull;
        ctl->launches += 1ull;
        ctl->inner_rounds += atomicAdd(&ctl->rounds_max, 0u);
        ctl->rounds_max = 0u;
        __threadfence();
        ctl->ticket = 0u;
    }
}

// ------------------------------------------------------------------------ tile kernel
// One CTA per tile; the tile plus a one-cell halo (faces only) is staged in shared memory;
// up to R rounds of the local-minimum test run on-chip. SYNC = false: asynchronous in-place
// updates (fig:a1c1pe semantics inside the tile); SYNC = true: the two
// barriers of fig:s1c1pe, private new_s/new_t then commit.
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

    // stage tile + face halo (slots with more than one coordinate outside are never read)
    for (int i = tid; i < NSLOT; i += NT) {
        const int lx = i % SX - 1, ly = (i / SX) % SY - 1, lz = (NDIM == 3) ? i / SXY - 1 : 0;
        const int out = (lx < 0 || lx >= TX) + (ly < 0 || ly >= TY) + ((NDIM == 3) && (lz < 0 || lz >= TZ));
        if (out <= 1) S[i] = ld_word(P, x0 + lx, y0 + ly, z0 + lz);
    }

    // owned cells of this thread: i = tid + k*NT
    unsigned long long wreg[CPT];
    uint32_t nreg[CPT];
    uint32_t valid = 0;
    const unsigned long long wlim = *(volatile unsigned long long*)&P.ctl->wlim;
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        const int i = tid + k * NT;
        const int lx = i % TX, ly = (i / TX) % TY, lz = i / (TX * TY);
        const int gx = x0 + lx, gy = y0 + ly, gz = z0 + lz;
        const bool v = gx < g.nx && gy < g.ny && (NDIM == 2 || gz < g.nz);
        nreg[k] = 0;
        if (v) {
            valid |= 1u << k;
            const size_t gi = NDIM == 2 ? (size_t)gy * g.nx + gx : ((size_t)gz * g.ny + gy) * g.nx + gx;
            nreg[k] = P.cnt[gi];
        }
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
    const uint32_t key0 = P.key0, key1 = P.key1;

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
            const int gx = x0 + lx, gy = y0 + ly, gz = z0 + lz;
            const unsigned long long cid = NDIM == 2
                ? (unsigned long long)(gy + g.y0) * g.nx + gx
                : ((unsigned long long)(gz + g.z0) * g.NY + gy) * g.nx + gx;
            const FireOut o = fire(w, ones, Z, nreg[k], cid, g.SH, thr, lr, key0, key1, P.inv_lambda,
                                   P.tie_bits, P.do_hash);
            hacc += o.h;
            flips += o.flip;
            ++fired;
            nreg[k] += 1;
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

    // write back the owned cells that changed; count cells still active
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
            P.cnt[gi] = nreg[k];
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

// ------------------------------------------------------------ tile kernel, compacted
// Same method and semantics as tile_kernel<..., SYNC=false>, organised for SIMT efficiency:
// per round every warp (i) tests its 512 cells against the current words — the test is a
// 32-bit compare of the high halves, with a full 64-bit compare only on a high-half tie —
// (ii) compacts the eligible cells into a warp-private queue with __ballot_sync, and
// (iii) fires them with all 32 lanes busy (Philox + NLOG + hash are ~90 % of the work; in
// the uncompacted kernel they ran with ~10 % of the lanes active).
// Correctness of firing after compaction: a queued cell c was a local minimum when
// tested; its word cannot change until it fires, so no neighbour can pass its own test
// (it would need a word below c's) — c's neighbourhood is frozen until c fires.
template <int NDIM, int TX, int TY, int TZ, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) tile2_kernel(const KParams P) {
    constexpr int SX = TX + 2, SY = TY + 2, SZ = (NDIM == 3) ? TZ + 2 : 1;
    constexpr int NSLOT = SX * SY * SZ;
    constexpr int NCELL = TX * TY * TZ;
    constexpr int NW = NT / 32;
    constexpr int CPW = NCELL / NW;        // cells per warp
    constexpr int JPL = CPW / 32;          // cells per lane
    static_assert(NCELL % NT == 0 && CPW % 32 == 0, "tile/block mismatch");
    constexpr int Z = 2 * NDIM;
    constexpr int SXY = SX * SY;

    if (*(volatile unsigned int*)&P.ctl->done) return;

    extern __shared__ __align__(16) unsigned long long smem[];
    unsigned long long* S = smem;                                   // NSLOT words
    unsigned long long* lr = S + NSLOT;                             // 512
    unsigned long long* thr = lr + 512;                             // 16
    unsigned long long* red = thr + 16;                             // NW
    unsigned int* Nc = (unsigned int*)(red + NW);                   // NCELL counters
    unsigned short* Q = (unsigned short*)(Nc + NCELL);              // NW * CPW queue

    const Geo& g = P.g;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int bt = blockIdx.x;
    const int tx = bt % P.tiles_x;
    const int ty = (bt / P.tiles_x) % P.tiles_y;
    const int tz = bt / (P.tiles_x * P.tiles_y);
    const int x0 = tx * TX, y0 = ty * TY, z0 = tz * TZ;
    const bool full_tile = x0 + TX <= g.nx && y0 + TY <= g.ny && (NDIM == 2 || z0 + TZ <= g.nz);

    for (int i = tid; i < 512; i += NT) lr[i] = P.lr[i];
    if (tid < 16) thr[tid] = tid < 14 ? P.thr[tid] : 0ull;
    for (int i = tid; i < NSLOT; i += NT) {
        const int lx = i % SX - 1, ly = (i / SX) % SY - 1, lz = (NDIM == 3) ? i / SXY - 1 : 0;
        const int out = (lx < 0 || lx >= TX) + (ly < 0 || ly >= TY) + ((NDIM == 3) && (lz < 0 || lz >= TZ));
        if (out <= 1) S[i] = ld_word(P, x0 + lx, y0 + ly, z0 + lz);
    }
    for (int o = tid; o < NCELL; o += NT) {
        const int lx = o % TX, ly = (o / TX) % TY, lz = o / (TX * TY);
        const int gx = x0 + lx, gy = y0 + ly, gz = z0 + lz;
        unsigned int nv = 0;
        if (gx < g.nx && gy < g.ny && (NDIM == 2 || gz < g.nz)) {
            const size_t gi = NDIM == 2 ? (size_t)gy * g.nx + gx : ((size_t)gz * g.ny + gy) * g.nx + gx;
            nv = P.cnt[gi];
        }
        Nc[o] = nv;
    }
    __syncthreads();

    volatile unsigned long long* VS = S;
    const volatile unsigned int* VH = (const volatile unsigned int*)S;   // VH[2s+1] = high half of S[s]
    const unsigned long long wlim = *(volatile unsigned long long*)&P.ctl->wlim;
    unsigned short* q = Q + warp * CPW;
    const int wbase = warp * CPW;
    unsigned long long fired = 0, flips = 0, tested = 0, hacc = 0;
    unsigned int rounds = 0;

    for (int r = 0; r < P.rounds; ++r) {
        // (i)+(ii): test and compact
        int cnt = 0;
#pragma unroll 4
        for (int j = 0; j < JPL; ++j) {
            const int o = wbase + lane + 32 * j;
            const int lx = o % TX, ly = (o / TX) % TY, lz = o / (TX * TY);
            const int s = (lz + (NDIM == 3)) * SXY + (ly + 1) * SX + lx + 1;
            bool e = false;
            const unsigned long long w = VS[s];
            bool valid = full_tile || (x0 + lx < g.nx && y0 + ly < g.ny && (NDIM == 2 || z0 + lz < g.nz));
            if (valid && w < wlim) {
                ++tested;
                const unsigned int oh = (unsigned int)(w >> 32);
                const unsigned int a = VH[2 * (s - 1) + 1], b = VH[2 * (s + 1) + 1];
                const unsigned int c = VH[2 * (s - SX) + 1], d = VH[2 * (s + SX) + 1];
                bool lt = oh < a && oh < b && oh < c && oh < d;
                bool gt = oh > a || oh > b || oh > c || oh > d;
                if (NDIM == 3) {
                    const unsigned int ee = VH[2 * (s - SXY) + 1], ff = VH[2 * (s + SXY) + 1];
                    lt = lt && oh < ee && oh < ff;
                    gt = gt || oh > ee || oh > ff;
                }
                if (lt) {
                    e = true;
                } else if (!gt) {   // a tie in the high halves: decide on the full words
                    e = w < VS[s - 1] && w < VS[s + 1] && w < VS[s - SX] && w < VS[s + SX];
                    if (NDIM == 3) e = e && w < VS[s - SXY] && w < VS[s + SXY];
                }
            }
            const unsigned int m = __ballot_sync(0xffffffffu, e);
            if (e) q[cnt + __popc(m & ((1u << lane) - 1u))] = (unsigned short)o;
            cnt += __popc(m);
        }
        __syncwarp();
        // (iii): fire the queued cells with the whole warp
        for (int i = lane; i < cnt; i += 32) {
            const int o = q[i];
            const int lx = o % TX, ly = (o / TX) % TY, lz = o / (TX * TY);
            const int s = (lz + (NDIM == 3)) * SXY + (ly + 1) * SX + lx + 1;
            const unsigned long long w = VS[s];
            const volatile unsigned int* VL = (const volatile unsigned int*)S;
            uint32_t ones = (VL[2 * (s - 1)] & 1u) + (VL[2 * (s + 1)] & 1u) + (VL[2 * (s - SX)] & 1u) +
                            (VL[2 * (s + SX)] & 1u);
            if (NDIM == 3) ones += (VL[2 * (s - SXY)] & 1u) + (VL[2 * (s + SXY)] & 1u);
            const int gx = x0 + lx, gy = y0 + ly, gz = z0 + lz;
            const unsigned long long cid = NDIM == 2
                ? (unsigned long long)(gy + g.y0) * g.nx + gx
                : ((unsigned long long)(gz + g.z0) * g.NY + gy) * g.nx + gx;
            const unsigned int k = Nc[o];
            const FireOut f = fire(w, ones, Z, k, cid, g.SH, thr, lr, P.key0, P.key1, P.inv_lambda,
                                   P.tie_bits, P.do_hash);
            VS[s] = f.wnew;
            Nc[o] = k + 1;
            hacc += f.h;
            flips += f.flip;
            ++fired;
        }
        ++rounds;
        if (__syncthreads_count(cnt > 0) == 0) break;
    }

    unsigned long long active = 0;
    for (int o = tid; o < NCELL; o += NT) {
        const int lx = o % TX, ly = (o / TX) % TY, lz = o / (TX * TY);
        const int gx = x0 + lx, gy = y0 + ly, gz = z0 + lz;
        if (gx < g.nx && gy < g.ny && (NDIM == 2 || gz < g.nz)) {
            const size_t gi = NDIM == 2 ? (size_t)gy * g.nx + gx : ((size_t)gz * g.ny + gy) * g.nx + gx;
            const unsigned long long w = S[(lz + (NDIM == 3)) * SXY + (ly + 1) * SX + lx + 1];
            P.words[gi] = w;
            P.cnt[gi] = Nc[o];
            active += w < wlim;
        }
    }
    const unsigned long long s_act = block_sum<NT>(active, red);
    const unsigned long long s_fir = block_sum<NT>(fired, red);
    const unsigned long long s_flp = block_sum<NT>(flips, red);
    const unsigned long long s_tst = block_sum<NT>(tested, red);
    const unsigned long long s_hsh = block_sum<NT>(hacc, red);
    if (tid == 0) finish_launch(P.ctl, s_act, s_fir, s_flp, s_tst, s_hsh, rounds);
}

// ------------------------------------------------------------ persistent TMA tile kernel
// tile2's rounds inside a persistent CTA that walks the tiles (tile = blockIdx.x + k*gridDim.x).
// Staging of a full tile: the tile's own rows of words and counters arrive by TMA bulk
// copies (cp.async.bulk, one mbarrier, ~48 KB in flight per CTA: no other CTA writes these
// rows, so a bulk copy is safe); the face halo — words other CTAs may be updating in place —
// is read with ordinary 8-byte loads (single-copy atomic, so a (t, s) pair is never torn).
// Write-back uses 16-byte vector stores. Smem row stride TX+4 puts the interior of every
// row on a 16-byte boundary. Ragged / odd-width tiles take the generic per-word path.
__device__ __forceinline__ unsigned long long ld_word1(const KParams& P, int gx, int gy, int gz) {
    const Geo& g = P.g;
    const int x = wrap1(gx, g.nx);
    if (g.ndim == 2) {
        if (!g.sharded) return P.words[(size_t)wrap1(gy, g.ny) * g.nx + x];
        if (gy < 0) return P.halo_lo[x];
        if (gy >= g.ny) return P.halo_hi[x];
        return P.words[(size_t)gy * g.nx + x];
    }
    const int y = wrap1(gy, g.ny);
    if (!g.sharded) return P.words[((size_t)wrap1(gz, g.nz) * g.ny + y) * g.nx + x];
    if (gz < 0) return P.halo_lo[(size_t)y * g.nx + x];
    if (gz >= g.nz) return P.halo_hi[(size_t)y * g.nx + x];
    return P.words[((size_t)gz * g.ny + y) * g.nx + x];
}

template <int NDIM, int TX, int TY, int TZ, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) tile3_kernel(const KParams P) {
    constexpr int SX = TX + 4, SY = TY + 2, SZ = (NDIM == 3) ? TZ + 2 : 1;
    constexpr int SXY = SX * SY;
    constexpr int NSLOT = SXY * SZ;
    constexpr int NCELL = TX * TY * TZ;
    constexpr int NROWS = TY * TZ;
    constexpr int NW = NT / 32;
    constexpr int CPW = NCELL / NW;
    constexpr int JPL = CPW / 32;
    constexpr int Z = 2 * NDIM;
    constexpr int NHALO = NDIM == 2 ? 2 * (TX + TY) : 2 * (TX * TY + TX * TZ + TY * TZ);
    static_assert(NCELL % NT == 0 && CPW % 32 == 0 && TX % 4 == 0, "tile/block mismatch");

    if (*(volatile unsigned int*)&P.ctl->done) return;

    extern __shared__ __align__(128) unsigned long long smem[];
    unsigned long long* S = smem;                                   // NSLOT words
    unsigned long long* lr = S + NSLOT;                             // 512
    unsigned long long* thr = lr + 512;                             // 16
    unsigned long long* red = thr + 16;                             // NW
    unsigned long long* bar = red + NW;                             // 1 (+1 pad)
    unsigned int* Nc = (unsigned int*)(bar + 2);                    // NCELL counters (16-B aligned)
    unsigned short* Q = (unsigned short*)(Nc + NCELL);              // NW * CPW queue

    const Geo& g = P.g;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < 512; i += NT) lr[i] = P.lr[i];
    if (tid < 16) thr[tid] = tid < 14 ? P.thr[tid] : 0ull;
    if (tid == 0) mbar_init(bar, 1);
    __syncthreads();

    auto slot = [](int lx, int ly, int lz) { return (lz + (NDIM == 3)) * SXY + (ly + 1) * SX + lx + 2; };
    volatile unsigned long long* VS = S;
    const volatile unsigned int* VH = (const volatile unsigned int*)S;   // [2s+1]: high half, [2s]: low half
    const unsigned long long wlim = *(volatile unsigned long long*)&P.ctl->wlim;
    unsigned short* q = Q + warp * CPW;
    const int wbase = warp * CPW;
    const int ntiles = P.tiles_x * P.tiles_y * P.tiles_z;
    const bool vec_ok = (g.nx % 4) == 0;
    unsigned long long fired = 0, flips = 0, tested = 0, hacc = 0, active = 0;
    unsigned int rounds_max = 0;
    uint32_t parity = 0;

    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int tx = tile % P.tiles_x;
        const int ty = (tile / P.tiles_x) % P.tiles_y;
        const int tz = tile / (P.tiles_x * P.tiles_y);
        const int x0 = tx * TX, y0 = ty * TY, z0 = tz * TZ;
        const bool full = x0 + TX <= g.nx && y0 + TY <= g.ny && (NDIM == 2 || z0 + TZ <= g.nz);
        const bool fast = full && vec_ok;

        // ------------------------------------------------ stage
        if (fast) {
            if (warp == 0) {
                if (lane == 0) mbar_arrive_expect_tx(bar, (uint32_t)NROWS * TX * 12u);
                __syncwarp();
                fence_proxy_async();
                for (int row = lane; row < NROWS; row += 32) {
                    const int ly = row % TY, lz = row / TY;
                    const size_t gi = NDIM == 2 ? (size_t)(y0 + ly) * g.nx + x0
                                                : ((size_t)(z0 + lz) * g.ny + (y0 + ly)) * g.nx + x0;
                    bulk_g2s(&S[slot(0, ly, lz)], P.words + gi, TX * 8, bar);
                    bulk_g2s(&Nc[row * TX], P.cnt + gi, TX * 4, bar);
                }
            }
            for (int h = tid; h < NHALO; h += NT) {
                int lx, ly, lz = 0;
                if (NDIM == 2) {
                    if (h < TX) { lx = h; ly = -1; }
                    else if (h < 2 * TX) { lx = h - TX; ly = TY; }
                    else if (h < 2 * TX + TY) { lx = -1; ly = h - 2 * TX; }
                    else { lx = TX; ly = h - 2 * TX - TY; }
                } else {
                    int r = h;
                    if (r < 2 * TX * TY) { lz = r < TX * TY ? -1 : TZ; r %= TX * TY; lx = r % TX; ly = r / TX; }
                    else if ((r -= 2 * TX * TY) < 2 * TX * TZ) {
                        ly = r < TX * TZ ? -1 : TY; r %= TX * TZ; lx = r % TX; lz = r / TX;
                    } else {
                        r -= 2 * TX * TZ;
                        lx = r < TY * TZ ? -1 : TX; r %= TY * TZ; ly = r % TY; lz = r / TY;
                    }
                }
                S[slot(lx, ly, lz)] = ld_word1(P, x0 + lx, y0 + ly, z0 + lz);
            }
            mbar_wait(bar, parity);
            parity ^= 1u;
        } else {
            for (int i = tid; i < NSLOT; i += NT) {
                const int lx = i % SX - 2, ly = (i / SX) % SY - 1, lz = (NDIM == 3) ? i / SXY - 1 : 0;
                if (lx < -1 || lx > TX) continue;
                const int out = (lx < 0 || lx >= TX) + (ly < 0 || ly >= TY) + ((NDIM == 3) && (lz < 0 || lz >= TZ));
                if (out <= 1) S[i] = ld_word(P, x0 + lx, y0 + ly, z0 + lz);
            }
            for (int o = tid; o < NCELL; o += NT) {
                const int lx = o % TX, ly = (o / TX) % TY, lz = o / (TX * TY);
                const int gx = x0 + lx, gy = y0 + ly, gz = z0 + lz;
                unsigned int nv = 0;
                if (gx < g.nx && gy < g.ny && (NDIM == 2 || gz < g.nz)) {
                    const size_t gi = NDIM == 2 ? (size_t)gy * g.nx + gx : ((size_t)gz * g.ny + gy) * g.nx + gx;
                    nv = P.cnt[gi];
                }
                Nc[o] = nv;
            }
        }
        __syncthreads();

        // ------------------------------------------------ rounds
        // Lane `lane` of warp `warp` owns cells o_j = warp*CPW + lane + 32 j. With FASTMAP the
        // slot of o_j is s_0 + const(j): all shared-memory addresses become immediates.
        constexpr bool FASTMAP = (TX % 32 == 0) && (CPW % TX == 0) && (TY % (CPW / TX == 0 ? 1 : CPW / TX) == 0);
        constexpr int LPR = TX / 32 > 0 ? TX / 32 : 1;                  // lane-groups per row
        int s0 = 0;
        if (FASTMAP) {
            const int row0 = warp * (CPW / TX);
            s0 = slot(lane, row0 % TY, row0 / TY);
        }
        unsigned int rounds = 0;
        for (int r = 0; r < P.rounds; ++r) {
            uint32_t emask = 0, amask = 0;
#pragma unroll
            for (int j = 0; j < JPL; ++j) {
                int s;
                bool valid = true;
                if (FASTMAP) {
                    s = s0 + (j / LPR) * SX + 32 * (j % LPR);
                    if (!full) {
                        const int o = wbase + lane + 32 * j;
                        const int lx = o % TX, ly = (o / TX) % TY, lz = o / (TX * TY);
                        valid = x0 + lx < g.nx && y0 + ly < g.ny && (NDIM == 2 || z0 + lz < g.nz);
                    }
                } else {
                    const int o = wbase + lane + 32 * j;
                    const int lx = o % TX, ly = (o / TX) % TY, lz = o / (TX * TY);
                    s = slot(lx, ly, lz);
                    valid = full || (x0 + lx < g.nx && y0 + ly < g.ny && (NDIM == 2 || z0 + lz < g.nz));
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
                    emask |= (uint32_t)e << j;
                }
                amask |= (uint32_t)act << j;
            }
            tested += __popc(amask);
            // compaction: warp-exclusive scan of the per-lane counts
            const int mine = __popc(emask);
            int incl = mine;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += v;
            }
            const int cnt = __shfl_sync(0xffffffffu, incl, 31);
            int pos = incl - mine;
            while (emask) {
                const int j = __ffs(emask) - 1;
                emask &= emask - 1u;
                q[pos++] = (unsigned short)(wbase + lane + 32 * j);
            }
            __syncwarp();
            for (int i = lane; i < cnt; i += 32) {
                const int o = q[i];
                const int lx = o % TX, ly = (o / TX) % TY, lz = o / (TX * TY);
                const int s = slot(lx, ly, lz);
                const unsigned long long w = VS[s];
                uint32_t ones = (VH[2 * (s - 1)] & 1u) + (VH[2 * (s + 1)] & 1u) + (VH[2 * (s - SX)] & 1u) +
                                (VH[2 * (s + SX)] & 1u);
                if (NDIM == 3) ones += (VH[2 * (s - SXY)] & 1u) + (VH[2 * (s + SXY)] & 1u);
                const int gx = x0 + lx, gy = y0 + ly, gz = z0 + lz;
                const unsigned long long cid = NDIM == 2
                    ? (unsigned long long)(gy + g.y0) * g.nx + gx
                    : ((unsigned long long)(gz + g.z0) * g.NY + gy) * g.nx + gx;
                const unsigned int k = Nc[o];
                const FireOut f = fire(w, ones, Z, k, cid, g.SH, thr, lr, P.key0, P.key1, P.inv_lambda,
                                       P.tie_bits, P.do_hash);
                VS[s] = f.wnew;
                Nc[o] = k + 1;
                hacc += f.h;
                flips += f.flip;
                ++fired;
            }
            ++rounds;
            if (__syncthreads_count(cnt > 0) == 0) break;
        }
        rounds_max = rounds > rounds_max ? rounds : rounds_max;
        __syncthreads();

        // ------------------------------------------------ write back
        if (fast) {
            for (int idx = tid; idx < NROWS * (TX / 2); idx += NT) {
                const int row = idx / (TX / 2), m2 = 2 * (idx % (TX / 2));
                const int ly = row % TY, lz = row / TY;
                const size_t gi = NDIM == 2 ? (size_t)(y0 + ly) * g.nx + x0
                                            : ((size_t)(z0 + lz) * g.ny + (y0 + ly)) * g.nx + x0;
                const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(&S[slot(m2, ly, lz)]);
                *reinterpret_cast<ulonglong2*>(P.words + gi + m2) = v;
                active += (v.x < wlim) + (v.y < wlim);
            }
            for (int idx = tid; idx < NROWS * (TX / 4); idx += NT) {
                const int row = idx / (TX / 4), m4 = 4 * (idx % (TX / 4));
                const int ly = row % TY, lz = row / TY;
                const size_t gi = NDIM == 2 ? (size_t)(y0 + ly) * g.nx + x0
                                            : ((size_t)(z0 + lz) * g.ny + (y0 + ly)) * g.nx + x0;
                *reinterpret_cast<uint4*>(P.cnt + gi + m4) = *reinterpret_cast<const uint4*>(&Nc[row * TX + m4]);
            }
        } else {
            for (int o = tid; o < NCELL; o += NT) {
                const int lx = o % TX, ly = (o / TX) % TY, lz = o / (TX * TY);
                const int gx = x0 + lx, gy = y0 + ly, gz = z0 + lz;
                if (gx < g.nx && gy < g.ny && (NDIM == 2 || gz < g.nz)) {
                    const size_t gi = NDIM == 2 ? (size_t)gy * g.nx + gx : ((size_t)gz * g.ny + gy) * g.nx + gx;
                    const unsigned long long w = S[slot(lx, ly, lz)];
                    P.words[gi] = w;
                    P.cnt[gi] = Nc[o];
                    active += w < wlim;
                }
            }
        }
        __syncthreads();   // smem is rewritten by the next tile's staging
    }
    const unsigned long long s_act = block_sum<NT>(active, red);
    const unsigned long long s_fir = block_sum<NT>(fired, red);
    const unsigned long long s_flp = block_sum<NT>(flips, red);
    const unsigned long long s_tst = block_sum<NT>(tested, red);
    const unsigned long long s_hsh = block_sum<NT>(hacc, red);
    if (tid == 0) finish_launch(P.ctl, s_act, s_fir, s_flp, s_tst, s_hsh, rounds_max);
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
    unsigned int* ns = (unsigned int*)(pend + (SYNC ? N : 0));   // N counters
    const int tid = threadIdx.x;
    const int Z = 2 * g.ndim;
    for (int i = tid; i < 512; i += NT) lr[i] = P.lr[i];
    if (tid < 16) thr[tid] = tid < 14 ? P.thr[tid] : 0ull;
    for (int i = tid; i < N; i += NT) {
        S[i] = P.words[i];
        ns[i] = P.cnt[i];
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
            if (g.ndim == 3) {
                const int zm = i + ((z == 0 ? g.nz - 1 : z - 1) - z) * pl;
                const int zp = i + ((z == g.nz - 1 ? 0 : z + 1) - z) * pl;
                const unsigned long long e = VS[zm], f = VS[zp];
                ok = ok && w < e && w < f;
                ones += (uint32_t)(e & 1ull) + (uint32_t)(f & 1ull);
            }
            if (!ok) continue;
            const FireOut o = fire(w, ones, Z, ns[i], (unsigned long long)i, g.SH, thr, lr, P.key0, P.key1,
                                   P.inv_lambda, P.tie_bits, P.do_hash);
            hacc += o.h;
            flips += o.flip;
            ++fired;
            ns[i] += 1;
            any = 1;
            if (SYNC) pend[i] = o.wnew;   // private new_s/new_t (word 0 never occurs: t >= 1)
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
        P.cnt[i] = ns[i];
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
__global__ void init_kernel(unsigned long long* __restrict__ words, unsigned int* __restrict__ cnt, Geo g,
                            const unsigned long long* __restrict__ lr_g, uint32_t key0, uint32_t key1,
                            unsigned long long thr_init, unsigned long long inv_lambda, int tie_bits,
                            unsigned long long n_local) {
    __shared__ unsigned long long lr[512];
    for (int i = threadIdx.x; i < 512; i += blockDim.x) lr[i] = lr_g[i];
    __syncthreads();
    const unsigned long long plane = (unsigned long long)g.nx * g.ny;
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n_local;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long x = i % g.nx;
        unsigned long long c, rank;
        if (g.ndim == 2) {
            const unsigned long long y = i / g.nx + g.y0;
            c = y * g.nx + x;
            rank = x + y;
        } else {
            const unsigned long long y = (i / g.nx) % g.ny, z = i / plane + g.z0;
            c = (z * g.NY + y) * g.nx + x;
            rank = x + y + z;
        }
        const u32x4 r = philox4x32_10(0u, (uint32_t)c, (uint32_t)(c >> 32), 1u, key0, key1);
        const unsigned long long sb = ((unsigned long long)r.x < thr_init) ? 0ull : 1ull;
        const unsigned long long t0 = delta_q32(r.y, r.z, lr, ACA_LN2_Q48, inv_lambda, tie_bits);
        words[i] = (t0 << g.SH) | (rank << 1) | sb;
        cnt[i] = 0u;
    }
}

// Repack (t, s) from host-provided spins / times into words (aca_set_state / aca_set_spins).
// Element i of the launch is shard-local cell base + i.
__global__ void pack_kernel(unsigned long long* __restrict__ words, const int8_t* __restrict__ spins,
                            const unsigned long long* __restrict__ times, Geo g, unsigned long long n,
                            unsigned long long base) {
    const unsigned long long plane = (unsigned long long)g.nx * g.ny;
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long li = base + i;
        const unsigned long long x = li % g.nx;
        unsigned long long rank;
        if (g.ndim == 2) rank = x + li / g.nx + g.y0;
        else rank = x + (li / g.nx) % g.ny + li / plane + g.z0;
        const unsigned long long w = words[i];
        const unsigned long long t = times ? times[i] : (w >> g.SH);
        const unsigned long long sb = spins ? (spins[i] > 0 ? 1ull : 0ull) : (w & 1ull);
        words[i] = (t << g.SH) | (rank << 1) | sb;
    }
}

// Unpack spins (int8) and times (u64) for the getters.
__global__ void unpack_kernel(const unsigned long long* __restrict__ words, int8_t* __restrict__ spins,
                              unsigned long long* __restrict__ times, int SH, unsigned long long n) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long w = words[i];
        if (spins) spins[i] = (w & 1ull) ? (int8_t)1 : (int8_t)-1;
        if (times) times[i] = w >> SH;
    }
}

// Statistics over the owned cells: B (bonds along +e_a), M, sum n, t_min, t_max.
struct StatAcc {
    long long bond, mag;
    unsigned long long arrivals, tmin, tmax;
};

template <int NT>
__global__ void __launch_bounds__(NT) stats_kernel(const KParams P, StatAcc* out, unsigned long long n_local) {
    const Geo& g = P.g;
    long long bond = 0, mag = 0;
    unsigned long long arr = 0, tmin = ~0ull, tmax = 0;
    const unsigned long long plane = (unsigned long long)g.nx * g.ny;
    for (unsigned long long i = blockIdx.x * (unsigned long long)NT + threadIdx.x; i < n_local;
         i += (unsigned long long)gridDim.x * NT) {
        const unsigned long long w = P.words[i];
        const int s = (w & 1ull) ? 1 : -1;
        const int x = (int)(i % g.nx);
        int y, z;
        if (g.ndim == 2) { y = (int)(i / g.nx); z = 0; }
        else { y = (int)((i / g.nx) % g.ny); z = (int)(i / plane); }
        int plus = ((ld_word(P, x + 1, y, z) & 1ull) ? 1 : -1) + ((ld_word(P, x, y + 1, z) & 1ull) ? 1 : -1);
        if (g.ndim == 3) plus += (ld_word(P, x, y, z + 1) & 1ull) ? 1 : -1;
        bond += s * plus;
        mag += s;
        arr += P.cnt[i];
        const unsigned long long t = w >> g.SH;
        tmin = t < tmin ? t : tmin;
        tmax = t > tmax ? t : tmax;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        bond += __shfl_xor_sync(0xffffffffu, bond, o);
        mag += __shfl_xor_sync(0xffffffffu, mag, o);
        arr += __shfl_xor_sync(0xffffffffu, arr, o);
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, tmin, o);
        const unsigned long long b = __shfl_xor_sync(0xffffffffu, tmax, o);
        tmin = a < tmin ? a : tmin;
        tmax = b > tmax ? b : tmax;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd((unsigned long long*)&out->bond, (unsigned long long)bond);
        atomicAdd((unsigned long long*)&out->mag, (unsigned long long)mag);
        atomicAdd(&out->arrivals, arr);
        atomicMin(&out->tmin, tmin);
        atomicMax(&out->tmax, tmax);
    }
}

}  // namespace aca
