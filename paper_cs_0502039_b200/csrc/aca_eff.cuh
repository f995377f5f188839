// aca_eff.cuh — time-only efficiency model of PAPER.md:1355-1442 on the GPU.
//
// For an Ising model next_t does not depend on the states, so whether a
// cell passes the test of fig:s1c1pe step 2 is decided by the local times alone. One
// iteration: every cell whose (t, c) is below every neighbour's (P6 order) draws its next
// increment; all tests see the previous iteration's times (ping-pong buffers). N0 per
// iteration is accumulated on the device; N0/N is the iteration's efficiency (PAPER.md:
// 1338-1353). Draw of iteration r: Philox ctr (r, c_lo, c_hi, TAG_EFF = 2); initial times from
// the P5 draw (0, c, 0, TAG_INIT = 1); laws as P3L. ndim 1 (n-circle), 2 (torus), 3.
//
// Bound: HBM streaming — per cell and iteration one 8-byte read (the neighbours' reads hit
// L1/L2) and one 8-byte write.
#pragma once
#include "aca_prim.cuh"
#include "nlog_tables.cuh"

namespace aca {

struct EffParams {
    int ndim;
    long long nx, ny, nz, N;
    unsigned long long mx, my;           // Lemire reciprocals ceil(2^64 / nx), ceil(2^64 / ny) (N < 2^32)
    uint32_t rk[20];
    unsigned long long inv_lambda;
    int law;
    int q;                               // neighbourhood degree (Eq. neiq): Manhattan radius
};

__global__ void __launch_bounds__(256) eff_init_kernel(unsigned long long* __restrict__ t, const EffParams P,
                                                       const unsigned long long* __restrict__ lr_g) {
    __shared__ unsigned long long lr[512];
    for (int i = threadIdx.x; i < 512; i += blockDim.x) lr[i] = lr_g[i];
    __syncthreads();
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < P.N; c += (long long)gridDim.x * blockDim.x) {
        const u32x4 r = philox4x32_10_rk(0u, (uint32_t)c, (uint32_t)((unsigned long long)c >> 32), 1u, P.rk);
        t[c] = delta_q32(r.y, r.z, lr, ACA_LN2_Q48, P.inv_lambda, 0, P.law);
    }
}

__device__ __forceinline__ bool lex_below(unsigned long long t, long long c, unsigned long long tn, long long n) {
    return t < tn || (t == tn && c < n);
}

template <int NDIM>
__global__ void __launch_bounds__(256) eff_round_kernel(const unsigned long long* __restrict__ tin,
                                                        unsigned long long* __restrict__ tout, const EffParams P,
                                                        const unsigned long long* __restrict__ lr_g, uint32_t round,
                                                        unsigned long long* __restrict__ fired) {
    __shared__ unsigned long long lr[512];
    __shared__ unsigned int red[8];
    for (int i = threadIdx.x; i < 512; i += blockDim.x) lr[i] = lr_g[i];
    __syncthreads();
    unsigned int n0 = 0;
    const long long nxy = P.nx * P.ny;
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < P.N; c += (long long)gridDim.x * blockDim.x) {
        const unsigned long long t = tin[c];
        const long long x = c % P.nx;
        const long long y = NDIM >= 2 ? (c / P.nx) % P.ny : 0;
        const long long z = NDIM == 3 ? c / nxy : 0;
        bool ok = true;
        const int q = P.q, qy = NDIM >= 2 ? q : 0, qz = NDIM == 3 ? q : 0;
        for (int dz = -qz; dz <= qz && ok; ++dz)
            for (int dy = -qy; dy <= qy && ok; ++dy)
                for (int dx = -q; dx <= q && ok; ++dx) {
                    const int dist = abs(dx) + abs(dy) + abs(dz);
                    if (dist == 0 || dist > q) continue;
                    const long long xx = ((x + dx) % P.nx + P.nx) % P.nx;
                    const long long yy = NDIM >= 2 ? ((y + dy) % P.ny + P.ny) % P.ny : 0;
                    const long long zz = NDIM == 3 ? ((z + dz) % P.nz + P.nz) % P.nz : 0;
                    const long long nb = (zz * P.ny + yy) * P.nx + xx;
                    if (nb != c) ok = lex_below(t, c, __ldg(tin + nb), nb);
                }
        unsigned long long tn = t;
        if (ok) {
            const u32x4 r = philox4x32_10_rk(round, (uint32_t)c, (uint32_t)((unsigned long long)c >> 32), 2u, P.rk);
            tn = t + delta_q32(r.y, r.z, lr, ACA_LN2_Q48, P.inv_lambda, 0, P.law);
            ++n0;
        }
        tout[c] = tn;
    }
    for (int o = 16; o > 0; o >>= 1) n0 += __shfl_xor_sync(0xffffffffu, n0, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = n0;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
        atomicAdd(fired + round, s);
    }
}

// n / d for n, d < 2^32 with M = ceil(2^64 / d) (Lemire, Kaser, Kurz 2019: exact for 32-bit n).
__device__ __forceinline__ uint32_t fdiv(uint32_t n, unsigned long long M) { return (uint32_t)__umul64hi(M, n); }

// Compacted iteration (N < 2^32): each warp takes chunks of 256 consecutive cells; every lane
// tests 8 cells (coalesced), copies the non-firing ones to the output, queues the firing ones
// (about 12 % in 2-D) in a per-warp list and the whole warp then draws their increments
// together (one Philox + law per lane instead of a divergent branch in most warps).
template <int NDIM>
__global__ void __launch_bounds__(256) eff_round_kernel_c(const unsigned long long* __restrict__ tin,
                                                          unsigned long long* __restrict__ tout, const EffParams P,
                                                          const unsigned long long* __restrict__ lr_g, uint32_t round,
                                                          unsigned long long* __restrict__ fired) {
    constexpr int J = 8;
    __shared__ unsigned long long lr[512];
    __shared__ unsigned int red[8];
    __shared__ uint32_t qc[8][32 * J];
    __shared__ unsigned long long qt[8][32 * J];
    for (int i = threadIdx.x; i < 512; i += blockDim.x) lr[i] = lr_g[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t nx = (uint32_t)P.nx, ny = (uint32_t)P.ny, nz = (uint32_t)P.nz, N = (uint32_t)P.N;
    const uint32_t nxy = nx * ny;
    const uint32_t nchunk = (N + 32 * J - 1) / (32 * J);
    unsigned int n0 = 0;
    for (uint32_t ch = blockIdx.x * 8 + warp; ch < nchunk; ch += gridDim.x * 8) {
        uint32_t fm = 0;
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const uint32_t c = ch * (32 * J) + lane + 32 * j;
            if (c >= N) continue;
            const unsigned long long t = tin[c];
            const uint32_t q1 = fdiv(c, P.mx);             // row index
            const uint32_t x = c - q1 * nx, row = c - x;
            const uint32_t xm = row + (x == 0 ? nx - 1 : x - 1), xp = row + (x == nx - 1 ? 0 : x + 1);
            bool ok = lex_below(t, c, __ldg(tin + xm), xm) && lex_below(t, c, __ldg(tin + xp), xp);
            if (NDIM >= 2) {
                const uint32_t q2 = fdiv(q1, P.my);         // plane index
                const uint32_t y = q1 - q2 * ny;
                const uint32_t ym = y == 0 ? c + (ny - 1) * nx : c - nx;
                const uint32_t yp = y == ny - 1 ? c - (ny - 1) * nx : c + nx;
                ok = ok && lex_below(t, c, __ldg(tin + ym), ym) && lex_below(t, c, __ldg(tin + yp), yp);
                if (NDIM == 3) {
                    const uint32_t z = q2;
                    const uint32_t zm = z == 0 ? c + (nz - 1) * nxy : c - nxy;
                    const uint32_t zp = z == nz - 1 ? c - (nz - 1) * nxy : c + nxy;
                    ok = ok && lex_below(t, c, __ldg(tin + zm), zm) && lex_below(t, c, __ldg(tin + zp), zp);
                }
            }
            if (ok) {
                fm |= 1u << j;
                qt[warp][lane + 32 * j] = t;   // the firing cell's time, for the draw phase
            } else {
                tout[c] = t;
            }
        }
        // compaction of the firing cells of this chunk
        const int mine = __popc(fm);
        int incl = mine;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += v;
        }
        const int cnt = __shfl_sync(0xffffffffu, incl, 31);
        int pos = incl - mine;
        unsigned long long tl[J];
        __syncwarp();
#pragma unroll
        for (int j = 0; j < J; ++j) tl[j] = qt[warp][lane + 32 * j];
        __syncwarp();
#pragma unroll
        for (int j = 0; j < J; ++j) {
            if ((fm >> j) & 1u) {
                qc[warp][pos] = ch * (32 * J) + lane + 32 * j;
                qt[warp][pos] = tl[j];
                ++pos;
            }
        }
        __syncwarp();
        for (int i = lane; i < cnt; i += 32) {
            const uint32_t c = qc[warp][i];
            const u32x4 r = philox4x32_10_rk(round, c, 0u, 2u, P.rk);
            tout[c] = qt[warp][i] + delta_q32(r.y, r.z, lr, ACA_LN2_Q48, P.inv_lambda, 0, P.law);
        }
        __syncwarp();
        n0 += (lane == 0) ? (unsigned int)cnt : 0u;
    }
    for (int o = 16; o > 0; o >>= 1) n0 += __shfl_xor_sync(0xffffffffu, n0, o);
    if (lane == 0) red[warp] = n0;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int w = 0; w < 8; ++w) s += red[w];
        atomicAdd(fired + round, s);
    }
}

// Row-streaming iteration for 2-D tori (N < 2^32, q = 1): a CTA of EFF_W threads owns a strip
// of EFF_W columns and a band of EFF_H rows; each thread owns one column and keeps the times
// of rows y-1, y, y+1 in registers, so every time is read from HBM once per iteration (plus
// two halo rows per band and two halo columns per row); the x-neighbours come from a
// double-buffered shared row (one barrier per row). Firing cells are queued per warp and drawn
// together every EFF_G rows by all warps at once (full lanes; a per-warp schedule would make
// every row's barrier wait for some warp's draws). Same results as eff_round_kernel_c.
constexpr int EFF_W = 256, EFF_H = 64, EFF_G = 8;

__global__ void __launch_bounds__(EFF_W) eff_round_kernel_2d(const unsigned long long* __restrict__ tin,
                                                              unsigned long long* __restrict__ tout, const EffParams P,
                                                              const unsigned long long* __restrict__ lr_g,
                                                              uint32_t round, unsigned long long* __restrict__ fired) {
    __shared__ unsigned long long lr[512];
    __shared__ unsigned long long row[2][EFF_W + 2];           // [0] left halo, [1..W] strip, [W+1] right halo
    __shared__ uint32_t qc[EFF_W / 32][32 * EFF_G];
    __shared__ unsigned long long qt[EFF_W / 32][32 * EFF_G];
    __shared__ unsigned int red[EFF_W / 32];
    for (int i = threadIdx.x; i < 512; i += blockDim.x) lr[i] = lr_g[i];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t nx = (uint32_t)P.nx, ny = (uint32_t)P.ny;
    const uint32_t x0 = blockIdx.x * EFF_W, yb = blockIdx.y * EFF_H;
    const uint32_t x = x0 + threadIdx.x;
    const bool inx = x < nx;
    const uint32_t ye = min(yb + EFF_H, ny);
    const uint32_t xl = x == 0 ? nx - 1 : x - 1, xr = x + 1 == nx ? 0 : x + 1;
    // the strip's neighbour columns: in the shared row when they fall inside the strip
    const bool l_in = inx && xl >= x0 && xl < x0 + EFF_W, r_in = inx && xr >= x0 && xr < x0 + EFF_W;
    const int l_slot = l_in ? (int)(xl - x0) + 1 : 0, r_slot = r_in ? (int)(xr - x0) + 1 : EFF_W + 1;
    // halo columns: the only outside neighbours a strip's threads can have
    const uint32_t xhl = x0 == 0 ? nx - 1 : x0 - 1;
    const uint32_t xhr = x0 + EFF_W < nx ? x0 + EFF_W : 0;
    auto row_of = [&](uint32_t yy) { return yy >= ny ? yy - ny : yy; };
    // registers: rows y-1, y, y+1 of the thread's column, and a prefetch ring of the next rows
    // (memory-level parallelism); the edge threads also prefetch their halo column
    constexpr int PF = 4;
    unsigned long long tu = 0, tm = 0, td = 0, pf[PF];
    if (inx) {
        const uint32_t yu = yb == 0 ? ny - 1 : yb - 1;
        tu = tin[(size_t)yu * nx + x];
        tm = tin[(size_t)yb * nx + x];
#pragma unroll
        for (int k = 0; k < PF; ++k) pf[k] = tin[(size_t)row_of(yb + 1 + k) * nx + x];
    }
    const bool hthr = threadIdx.x == 0 || threadIdx.x == EFF_W - 1;
    const uint32_t xh = threadIdx.x == 0 ? xhl : xhr;
    unsigned long long ph[PF + 1];
    if (hthr) {
#pragma unroll
        for (int k = 0; k <= PF; ++k) ph[k] = tin[(size_t)row_of(yb + k) * nx + xh];
    }
    unsigned int n0 = 0;
    int qn = 0;                                                      // warp queue length (uniform)
    int buf = 0;
    for (uint32_t y = yb; y < ye; ++y) {
        const uint32_t ydn = y + 1 == ny ? 0 : y + 1;
        const uint32_t yup = y == 0 ? ny - 1 : y - 1;
        if (inx) {
            td = pf[0];
#pragma unroll
            for (int k = 0; k < PF - 1; ++k) pf[k] = pf[k + 1];
            if (y + 1 + PF < ye + 1) pf[PF - 1] = tin[(size_t)row_of(y + 1 + PF) * nx + x];
        }
        row[buf][threadIdx.x + 1] = tm;
        if (hthr) {
            row[buf][threadIdx.x == 0 ? 0 : EFF_W + 1] = ph[0];
#pragma unroll
            for (int k = 0; k < PF; ++k) ph[k] = ph[k + 1];
            if (y + 1 + PF < ye) ph[PF] = tin[(size_t)row_of(y + 1 + PF) * nx + xh];
        }
        __syncthreads();
        bool ok = false;
        const uint32_t c = y * nx + x;
        if (inx) {
            const unsigned long long tl = row[buf][l_slot], tr = row[buf][r_slot];
            const uint32_t cl = y * nx + xl, cr = y * nx + xr, cu = yup * nx + x, cd = ydn * nx + x;
            ok = lex_below(tm, c, tl, cl) && lex_below(tm, c, tr, cr) && lex_below(tm, c, tu, cu) &&
                 lex_below(tm, c, td, cd);
            if (!ok) tout[c] = tm;
        }
        // queue the firing cells of this row (warp ballot)
        const unsigned int bm = __ballot_sync(0xffffffffu, ok);
        if (ok) {
            const int pos = qn + __popc(bm & ((1u << lane) - 1u));
            qc[warp][pos] = c;
            qt[warp][pos] = tm;
        }
        qn += __popc(bm);
        if ((y - yb) % EFF_G == EFF_G - 1 || y + 1 == ye) {          // all warps draw together (same row)
            __syncwarp();
            for (int i = lane; i < qn; i += 32) {
                const uint32_t cc = qc[warp][i];
                const u32x4 r = philox4x32_10_rk(round, cc, 0u, 2u, P.rk);
                tout[cc] = qt[warp][i] + delta_q32(r.y, r.z, lr, ACA_LN2_Q48, P.inv_lambda, 0, P.law);
            }
            n0 += lane == 0 ? (unsigned int)qn : 0u;
            qn = 0;
            __syncwarp();
        }
        tu = tm;
        tm = td;
        buf ^= 1;
    }
    for (int o = 16; o > 0; o >>= 1) n0 += __shfl_xor_sync(0xffffffffu, n0, o);
    if (lane == 0) red[warp] = n0;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long sacc = 0;
        for (int w = 0; w < EFF_W / 32; ++w) sacc += red[w];
        atomicAdd(fired + round, sacc);
    }
}

// ------------------------------------------------------------ fig:perfbl model (P11)
// The simplified many-cells-per-PE model with the lag bound of fig:perfbl
// (PAPER.md:1573-1605), docs/PRIMITIVES.md P11: a PE that selected a cell keeps it while blocked
// (fig:amcpoi Steps 2-3), so its pending event is a function of its counter
// alone. One CTA runs every round: the round reads the snapshot buffer hb[r & 1] and writes
// hb[(r + 1) & 1]; a block reduction gives the snapshot's minimum for the lag window.
struct PerfblParams {
    int px, py;
    unsigned long long E1, E2;          // category thresholds (floor((m-2)^2 2^32 / m^2), floor((m^2-4) 2^32 / m^2))
    unsigned long long lag;             // Q32, 0 = unbounded
    uint32_t rk[20];
    long long rounds;
    unsigned long long* hb;             // 2 x N
    unsigned int* n;                    // N
    unsigned long long* ups;            // rounds
};

template <int NT>
__global__ void __launch_bounds__(NT) perfbl_kernel(const PerfblParams A, const unsigned long long* __restrict__ lr_g) {
    __shared__ unsigned long long lr[512];
    __shared__ unsigned long long red[NT / 32];
    __shared__ unsigned long long bmin;
    for (int i = threadIdx.x; i < 512; i += NT) lr[i] = lr_g[i];
    const int N = A.px * A.py;
    for (int C = threadIdx.x; C < N; C += NT) {
        const u32x4 r = philox4x32_10_rk(0u, (uint32_t)C, 0u, 8u, A.rk);
        const uint64_t d = nlog_q32(((uint64_t)r.z << 32) | r.w, lr_g, ACA_LN2_Q48);
        A.hb[C] = d < 1 ? 1 : d;
        A.n[C] = 0u;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (long long r = 0; r < A.rounds; ++r) {
        const unsigned long long* hs = A.hb + (size_t)(r & 1) * N;
        unsigned long long* hn = A.hb + (size_t)((r + 1) & 1) * N;
        unsigned long long mn = ~0ull;
        for (int C = threadIdx.x; C < N; C += NT) mn = min(mn, hs[C]);
        for (int o = 16; o > 0; o >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        if (lane == 0) red[warp] = mn;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long m2 = red[0];
            for (int w = 1; w < NT / 32; ++w) m2 = min(m2, red[w]);
            bmin = m2;
        }
        __syncthreads();
        const unsigned long long hmin = bmin;
        unsigned long long cnt = 0;
        for (int C = threadIdx.x; C < N; C += NT) {
            const unsigned long long h = hs[C];
            unsigned long long out = h;
            if (!(A.lag && h - hmin >= A.lag)) {
                const unsigned int k = A.n[C];
                const u32x4 w = philox4x32_10_rk(k, (uint32_t)C, 0u, 7u, A.rk);
                const int cat = (unsigned long long)w.x < A.E1 ? 0 : ((unsigned long long)w.x < A.E2 ? 1 : 2);
                const int a = (int)(w.y >> 30), b = (a + 1 + (int)(((w.y & 0xffffu) * 3u) >> 16)) & 3;
                const int x = C % A.px, y = C / A.px;
                auto nbr = [&](int dir) {
                    const int xx = dir == 0 ? (x == 0 ? A.px - 1 : x - 1) : dir == 1 ? (x == A.px - 1 ? 0 : x + 1) : x;
                    const int yy = dir == 2 ? (y == 0 ? A.py - 1 : y - 1) : dir == 3 ? (y == A.py - 1 ? 0 : y + 1) : y;
                    return hs[yy * A.px + xx];
                };
                bool go = true;
                if (cat >= 1 && nbr(a) < h) go = false;
                if (cat == 2 && nbr(b) < h) go = false;
                if (go) {
                    const uint64_t d = nlog_q32(((uint64_t)w.z << 32) | w.w, lr, ACA_LN2_Q48);
                    out = h + (d < 1 ? 1 : d);
                    A.n[C] = k + 1;
                    ++cnt;
                }
            }
            hn[C] = out;
        }
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        __syncthreads();                                   // red[] is reused
        if (lane == 0) red[warp] = cnt;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long s2 = 0;
            for (int w = 0; w < NT / 32; ++w) s2 += red[w];
            A.ups[r] = s2;
        }
        __syncthreads();
    }
}

}  // namespace aca
