// aca_agg.cuh — the aggregated Poisson-stream algorithm of fig:amcpoi on
// the GPU (docs/PRIMITIVES.md P8).
//
// The 2-D torus is partitioned into m x m subarrays C (1 <= m <= 32; the paper's experiments use
// m = 12 and 24). One thread owns one subarray: its spins as m row masks, its cumulative-stream
// time T(C) (Q32) and arrival counter n(C). The thread processes its arrivals in order: draw
// (Philox, ctr (n, C, 0, tag)), choose the cell (Step 2), and if the cell has neighbours in
// other subarrays W(c), wait until (T(C), C) is below every (T(C'), C') of them (Step 3) —
// here: stop for this launch; the next launch retries. Then update the spin from the neighbour
// spins (Step 4) and advance T(C) (Step 5). Rows are published before times (store, fence,
// store; readers load the time, fence, then the row), so a neighbour that sees T(C') past its
// own time also sees every update of C' before it; a cell next to C is only ever changed at a
// time below C's (it waited for C), so the bits C reads are the states at its arrival time.
// The subarray with the smallest (T, C) is never blocked: every launch makes progress.
#pragma once
#include "aca_kernels.cuh"

namespace aca {

// State of a subarray C: its m spin rows rows[C m + j] (bit i set iff the cell (X m + i, Y m + j)
// is +1; m <= 32), its stream time T(C) (Q32) and its arrival counter n(C). A row is one 32-bit
// word, so a neighbour's read of a boundary bit is single-copy atomic.
struct AggParams {
    unsigned int* rows;           // [ntiles * m]
    unsigned long long* T;        // [ntiles], Q32
    unsigned int* n;              // [ntiles]
    int nx, ny, m, mx, my;        // lattice, subarray side, subarrays per row / column
    uint32_t rk[20];
    unsigned long long inv;       // floor(2^32 / (lambda m^2) + 0.5)
    unsigned long long Tend;
    uint32_t tag_e, tag_i;
    int budget;                   // arrivals per subarray per launch
    int do_hash;
    unsigned long long thr[10];
    unsigned long long thr_init;
};

struct AggAcc {
    unsigned long long arrivals, flips, hash, active, blocked;
};

// P5 spins of the subarray's cells, row by row
__device__ __forceinline__ void agg_init_rows(const AggParams& A, int C) {
    const int X = C % A.mx, Y = C / A.mx;
    for (int j = 0; j < A.m; ++j) {
        unsigned int row = 0;
        for (int i = 0; i < A.m; ++i) {
            const uint32_t c = (uint32_t)(Y * A.m + j) * (uint32_t)A.nx + (uint32_t)(X * A.m + i);
            const u32x4 r = philox4x32_10_rk(0u, c, 0u, 1u, A.rk);
            if ((unsigned long long)r.x >= A.thr_init) row |= 1u << i;
        }
        A.rows[(size_t)C * A.m + j] = row;
    }
}

__global__ void agg_init_kernel(const AggParams A, const unsigned long long* __restrict__ lr_g) {
    __shared__ unsigned long long lr[512];
    for (int i = threadIdx.x; i < 512; i += blockDim.x) lr[i] = lr_g[i];
    __syncthreads();
    const int NC = A.mx * A.my;
    for (int C = blockIdx.x * blockDim.x + threadIdx.x; C < NC; C += gridDim.x * blockDim.x) {
        agg_init_rows(A, C);
        const u32x4 r = philox4x32_10_rk(0u, (uint32_t)C, 0u, A.tag_i, A.rk);
        uint64_t q = nlog_q32(((uint64_t)r.y << 32) | r.z, lr, ACA_LN2_Q48);
        q = (__umul64hi(q, A.inv) << 32) | ((q * A.inv) >> 32);
        A.T[C] = q < 1 ? 1 : q;
        A.n[C] = 0u;
    }
}

__device__ __forceinline__ bool agg_below(unsigned long long t, int C, unsigned long long t2, int C2) {
    return t < t2 || (t == t2 && C < C2);
}

// Step 3 of fig:amcpoi for cell (i, j) of C: (T(C), C) below the subarrays holding its outside
// neighbours (W(c)).
__device__ __forceinline__ bool agg_may_go(const AggParams& A, volatile unsigned long long* VT, unsigned long long T,
                                           int C, int Cl, int Cr, int Cu, int Cd, int i, int j) {
    const int m = A.m;
    bool ok = true;
    if (i == 0 && Cl != C) ok = ok && agg_below(T, C, VT[Cl], Cl);
    if (i == m - 1 && Cr != C) ok = ok && agg_below(T, C, VT[Cr], Cr);
    if (j == 0 && Cu != C) ok = ok && agg_below(T, C, VT[Cu], Cu);
    if (j == m - 1 && Cd != C) ok = ok && agg_below(T, C, VT[Cd], Cd);
    return ok;
}
// number of +1 neighbours of cell (i, j) of C (periodic within the torus; the rows of the
// neighbouring subarrays for its outside neighbours) and its own spin bit
__device__ __forceinline__ uint32_t agg_ones(const AggParams& A, volatile unsigned int* VR, int C, int Cl, int Cr,
                                             int Cu, int Cd, int i, int j, uint32_t& sb) {
    const int m = A.m;
    const unsigned int rj = VR[(size_t)C * m + j];
    const uint32_t left = i > 0 ? (rj >> (i - 1)) & 1u : (VR[(size_t)Cl * m + j] >> (m - 1)) & 1u;
    const uint32_t right = i < m - 1 ? (rj >> (i + 1)) & 1u : VR[(size_t)Cr * m + j] & 1u;
    const uint32_t up = j > 0 ? (VR[(size_t)C * m + j - 1] >> i) & 1u : (VR[(size_t)Cu * m + m - 1] >> i) & 1u;
    const uint32_t down = j < m - 1 ? (VR[(size_t)C * m + j + 1] >> i) & 1u : (VR[(size_t)Cd * m] >> i) & 1u;
    sb = (rj >> i) & 1u;
    return left + right + up + down;
}

__global__ void __launch_bounds__(256) agg_round_kernel(const AggParams A, const unsigned long long* __restrict__ lr_g,
                                                        AggAcc* __restrict__ acc) {
    __shared__ unsigned long long lr[512];
    __shared__ unsigned long long red[5][8];
    for (int i = threadIdx.x; i < 512; i += blockDim.x) lr[i] = lr_g[i];
    __syncthreads();
    const int NC = A.mx * A.my;
    const int m = A.m;
    const unsigned long long mm = (unsigned long long)m * (unsigned long long)m;
    volatile unsigned long long* VT = A.T;
    volatile unsigned int* VR = A.rows;
    unsigned long long arr = 0, flips = 0, hsh = 0, active = 0, blocked = 0;
    for (int C = blockIdx.x * blockDim.x + threadIdx.x; C < NC; C += gridDim.x * blockDim.x) {
        const int X = C % A.mx, Y = C / A.mx;
        const int Cl = Y * A.mx + (X == 0 ? A.mx - 1 : X - 1), Cr = Y * A.mx + (X == A.mx - 1 ? 0 : X + 1);
        const int Cu = (Y == 0 ? A.my - 1 : Y - 1) * A.mx + X, Cd = (Y == A.my - 1 ? 0 : Y + 1) * A.mx + X;
        unsigned long long T = A.T[C];
        unsigned int k = A.n[C];
        for (int b = 0; b < A.budget && T < A.Tend; ++b) {
            const u32x4 r = philox4x32_10_rk(k, (uint32_t)C, 0u, A.tag_e, A.rk);
            const int l = (int)(((unsigned long long)r.w * mm) >> 32);   // Step 2: uniform cell of C (P8)
            const int i = l % m, j = l / m;
            if (!agg_may_go(A, VT, T, C, Cl, Cr, Cu, Cd, i, j)) { ++blocked; break; }
            __threadfence();                       // acquire: rows after the times we checked
            uint32_t sb;
            const uint32_t ones = agg_ones(A, VR, C, Cl, Cr, Cu, Cd, i, j, sb);   // Step 4
            const uint32_t flip = (unsigned long long)r.x < A.thr[ones + 5u * sb] ? 1u : 0u;
            uint64_t q = nlog_q32(((uint64_t)r.y << 32) | r.z, lr, ACA_LN2_Q48);
            q = (__umul64hi(q, A.inv) << 32) | ((q * A.inv) >> 32);
            q = q < 1 ? 1 : q;
            if (A.do_hash)
                hsh += ev_hash(r.w, T, ((unsigned long long)l << 1) ^ (unsigned long long)(sb ^ flip));
            if (flip) VR[(size_t)C * m + j] = VR[(size_t)C * m + j] ^ (1u << i);
            flips += flip;
            ++arr;
            ++k;
            T += q;                                // Step 5
            // publish: row, fence, time (release)
            A.n[C] = k;
            __threadfence();
            VT[C] = T;
        }
        active += T < A.Tend;
    }
    // block reduction of the counters
    unsigned long long v[5] = {arr, flips, hsh, active, blocked};
    for (int f = 0; f < 5; ++f)
        for (int o = 16; o > 0; o >>= 1) v[f] += __shfl_xor_sync(0xffffffffu, v[f], o);
    if ((threadIdx.x & 31) == 0)
        for (int f = 0; f < 5; ++f) red[f][threadIdx.x >> 5] = v[f];
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s[5] = {0, 0, 0, 0, 0};
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
            for (int f = 0; f < 5; ++f) s[f] += red[f][w];
        atomicAdd(&acc->arrivals, s[0]);
        atomicAdd(&acc->flips, s[1]);
        atomicAdd(&acc->hash, s[2]);
        atomicAdd(&acc->active, s[3]);
        atomicAdd(&acc->blocked, s[4]);
    }
}

// ------------------------------------------------------------------ modified BKL (P9)
// Kernel classes of row j (0 < j < m - 1) of a subarray: the number of +1 neighbours of every
// kernel cell by bit-sliced adders over the shifted row and its neighbour rows (kernel neighbours
// are inside the subarray), then the ten class masks M[idx(s, Sigma)], idx = ones + 5 [s = +1],
// restricted to the kernel columns (kcol: bits 1 .. m - 2).
__device__ __forceinline__ void bkl_row_classes(unsigned int S, unsigned int U, unsigned int D, unsigned int kcol,
                                                unsigned int* M) {
    const unsigned int L = S << 1, R = S >> 1;
    const unsigned int h1 = L ^ R, k1 = L & R, h2 = U ^ D, k2 = U & D;
    const unsigned int p0 = h1 ^ h2, c = h1 & h2;
    const unsigned int q0 = k1 ^ k2 ^ c, q1 = (k1 & k2) | (c & (k1 ^ k2));   // ones = p0 + 2 q0 + 4 q1
#pragma unroll
    for (int jj = 0; jj <= 4; ++jj) {
        const unsigned int e = ((jj & 1) ? p0 : ~p0) & ((jj & 2) ? q0 : ~q0) & ((jj & 4) ? q1 : ~q1) & kcol;
        M[jj] = e & ~S;           // s = -1
        M[jj + 5] = e & S;        // s = +1
    }
}
// total weight W = W0 + sum_k |Gamma_k| thr_k of subarray C (its own rows only)
__device__ __forceinline__ unsigned long long bkl_weight(const AggParams& A, volatile unsigned int* VR, int C,
                                                         unsigned int kcol, unsigned long long W0, unsigned int* cnt) {
    const int m = A.m;
#pragma unroll
    for (int q = 0; q < 10; ++q) cnt[q] = 0;
    for (int j = 1; j < m - 1; ++j) {
        unsigned int M[10];
        bkl_row_classes(VR[(size_t)C * m + j], VR[(size_t)C * m + j - 1], VR[(size_t)C * m + j + 1], kcol, M);
#pragma unroll
        for (int q = 0; q < 10; ++q) cnt[q] += __popc(M[q]);
    }
    unsigned long long W = W0;
#pragma unroll
    for (int q = 0; q < 10; ++q) W += (unsigned long long)cnt[q] * A.thr[q];
    return W;
}

__device__ __forceinline__ unsigned long long bkl_inv(double lambda, unsigned long long W) {
    return (unsigned long long)floor(18446744073709551616.0 / (lambda * (double)W) + 0.5);
}

struct BklExtra {
    double lambda;
    unsigned int kcol;            // kernel columns of a row (bits 1 .. m - 2)
    unsigned long long W0;        // |Gamma_0| 2^32 = (4m - 4) 2^32
};

__global__ void bkl_init_kernel(const AggParams A, const BklExtra E, const unsigned long long* __restrict__ lr_g) {
    __shared__ unsigned long long lr[512];
    for (int i = threadIdx.x; i < 512; i += blockDim.x) lr[i] = lr_g[i];
    __syncthreads();
    const int NC = A.mx * A.my;
    for (int C = blockIdx.x * blockDim.x + threadIdx.x; C < NC; C += gridDim.x * blockDim.x) {
        agg_init_rows(A, C);
        unsigned int cnt[10];
        const unsigned long long W = bkl_weight(A, A.rows, C, E.kcol, E.W0, cnt);
        const u32x4 r = philox4x32_10_rk(0u, (uint32_t)C, 0u, 6u, A.rk);
        const uint64_t q = nlog_q32(((uint64_t)r.z << 32) | r.w, lr, ACA_LN2_Q48);
        const unsigned long long inv = bkl_inv(E.lambda, W);
        const uint64_t d = (__umul64hi(q, inv) << 32) | ((q * inv) >> 32);
        A.T[C] = d < 1 ? 1 : d;
        A.n[C] = 0u;
    }
}

__global__ void __launch_bounds__(256) bkl_round_kernel(const AggParams A, const BklExtra E,
                                                        const unsigned long long* __restrict__ lr_g,
                                                        AggAcc* __restrict__ acc) {
    __shared__ unsigned long long lr[512];
    __shared__ unsigned long long red[5][8];
    for (int i = threadIdx.x; i < 512; i += blockDim.x) lr[i] = lr_g[i];
    __syncthreads();
    const int NC = A.mx * A.my;
    const int m = A.m;
    volatile unsigned long long* VT = A.T;
    volatile unsigned int* VR = A.rows;
    unsigned long long arr = 0, flips = 0, hsh = 0, active = 0, blocked = 0;
    for (int C = blockIdx.x * blockDim.x + threadIdx.x; C < NC; C += gridDim.x * blockDim.x) {
        const int X = C % A.mx, Y = C / A.mx;
        const int Cl = Y * A.mx + (X == 0 ? A.mx - 1 : X - 1), Cr = Y * A.mx + (X == A.mx - 1 ? 0 : X + 1);
        const int Cu = (Y == 0 ? A.my - 1 : Y - 1) * A.mx + X, Cd = (Y == A.my - 1 ? 0 : Y + 1) * A.mx + X;
        unsigned long long T = A.T[C];
        unsigned int k = A.n[C];
        for (int b = 0; b < A.budget && T < A.Tend; ++b) {
            const u32x4 r = philox4x32_10_rk(k, (uint32_t)C, 0u, 5u, A.rk);
            unsigned int cnt[10];
            const unsigned long long W = bkl_weight(A, VR, C, E.kcol, E.W0, cnt);
            const unsigned long long Xr = ((unsigned long long)r.x << 32) | r.y;
            const unsigned long long u = __umul64hi(Xr, W);
            int i, j;
            uint32_t sb, flip;
            if (u < E.W0) {   // boundary layer: the standard model, after waiting for W(c)
                const int bb = (int)(u >> 32);   // the bb-th cell of Gamma_0 in increasing l
                if (bb < m) { i = bb; j = 0; }
                else if (bb < m + 2 * (m - 2)) { j = 1 + (bb - m) / 2; i = ((bb - m) & 1) ? m - 1 : 0; }
                else { i = bb - m - 2 * (m - 2); j = m - 1; }
                if (!agg_may_go(A, VT, T, C, Cl, Cr, Cu, Cd, i, j)) { ++blocked; break; }
                __threadfence();
                const uint32_t ones = agg_ones(A, VR, C, Cl, Cr, Cu, Cd, i, j, sb);
                flip = (unsigned long long)(u & 0xffffffffull) < A.thr[ones + 5u * sb] ? 1u : 0u;
            } else {          // kernel: pick the class, then its cell; the cell flips
                unsigned long long o = u - E.W0;
                int kc = 0;
#pragma unroll
                for (int q = 0; q < 9; ++q) {
                    const unsigned long long Wk = (unsigned long long)cnt[kc] * A.thr[kc];
                    if (o < Wk) break;
                    o -= Wk;
                    ++kc;
                }
                unsigned int rr = (unsigned int)(o / A.thr[kc]);   // its rr-th cell in increasing l
                i = 0; j = 1;
                for (; j < m - 1; ++j) {
                    unsigned int M[10];
                    bkl_row_classes(VR[(size_t)C * m + j], VR[(size_t)C * m + j - 1], VR[(size_t)C * m + j + 1], E.kcol,
                                    M);
                    const unsigned int pc = __popc(M[kc]);
                    if (rr < pc) { i = (int)__fns(M[kc], 0, (int)rr + 1); break; }
                    rr -= pc;
                }
                sb = (VR[(size_t)C * m + j] >> i) & 1u;
                flip = 1u;
            }
            const int l = j * m + i;
            if (A.do_hash)
                hsh += ev_hash(r.w, T, ((unsigned long long)l << 1) ^ (unsigned long long)(sb ^ flip));
            if (flip) VR[(size_t)C * m + j] = VR[(size_t)C * m + j] ^ (1u << i);
            flips += flip;
            ++arr;
            ++k;
            const unsigned long long W2 = bkl_weight(A, VR, C, E.kcol, E.W0, cnt);
            const uint64_t q = nlog_q32(((uint64_t)r.z << 32) | r.w, lr, ACA_LN2_Q48);
            const unsigned long long inv = bkl_inv(E.lambda, W2);
            const uint64_t d = (__umul64hi(q, inv) << 32) | ((q * inv) >> 32);
            T += d < 1 ? 1 : d;
            A.n[C] = k;
            __threadfence();
            VT[C] = T;
        }
        active += T < A.Tend;
    }
    unsigned long long v[5] = {arr, flips, hsh, active, blocked};
    for (int f = 0; f < 5; ++f)
        for (int o = 16; o > 0; o >>= 1) v[f] += __shfl_xor_sync(0xffffffffu, v[f], o);
    if ((threadIdx.x & 31) == 0)
        for (int f = 0; f < 5; ++f) red[f][threadIdx.x >> 5] = v[f];
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long sm[5] = {0, 0, 0, 0, 0};
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
            for (int f = 0; f < 5; ++f) sm[f] += red[f][w];
        atomicAdd(&acc->arrivals, sm[0]);
        atomicAdd(&acc->flips, sm[1]);
        atomicAdd(&acc->hash, sm[2]);
        atomicAdd(&acc->active, sm[3]);
        atomicAdd(&acc->blocked, sm[4]);
    }
}

// Spins of the torus (int8, row-major) from the rows.
__global__ void agg_unpack_kernel(const AggParams A, int8_t* __restrict__ spins) {
    const long long N = (long long)A.nx * A.ny;
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < N; c += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(c % A.nx), y = (int)(c / A.nx);
        const int C = (y / A.m) * A.mx + x / A.m;
        spins[c] = (A.rows[(size_t)C * A.m + y % A.m] >> (x % A.m)) & 1u ? (int8_t)1 : (int8_t)-1;
    }
}

}  // namespace aca
