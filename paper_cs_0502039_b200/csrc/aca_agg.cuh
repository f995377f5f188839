// aca_agg.cuh — the aggregated Poisson-stream algorithm of fig:amcpoi on
// the GPU (docs/PRIMITIVES.md P8).
//
// The 2-D torus is partitioned into m x m subarrays C (m = 1, 2, 4, 8). One thread owns one
// subarray: its m^2 spins as a bit mask (bit l = j m + i set iff s = +1), its cumulative-stream
// time T(C) (Q32) and arrival counter n(C). The thread processes its arrivals in order: draw
// (Philox, ctr (n, C, 0, tag)), choose the cell (Step 2), and if the cell has neighbours in
// other subarrays W(c), wait until (T(C), C) is below every (T(C'), C') of them (Step 3) —
// here: stop for this launch; the next launch retries. Then update the spin from the neighbour
// spins (Step 4) and advance T(C) (Step 5). Masks are published before times (store, fence,
// store; readers load the time, fence, then the mask), so a neighbour that sees T(C') past its
// own time also sees every update of C' before it; a cell next to C is only ever changed at a
// time below C's (it waited for C), so the mask bits C reads are the states at its arrival time.
// The subarray with the smallest (T, C) is never blocked: every launch makes progress.
#pragma once
#include "aca_kernels.cuh"

namespace aca {

struct AggParams {
    unsigned long long* mask;     // [ntiles]
    unsigned long long* T;        // [ntiles], Q32
    unsigned int* n;              // [ntiles]
    int nx, ny, m, lg, mx, my;    // lattice, subarray side, log2(m^2), subarrays per row / column
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

__global__ void agg_init_kernel(const AggParams A, const unsigned long long* __restrict__ lr_g) {
    __shared__ unsigned long long lr[512];
    for (int i = threadIdx.x; i < 512; i += blockDim.x) lr[i] = lr_g[i];
    __syncthreads();
    const int NC = A.mx * A.my;
    for (int C = blockIdx.x * blockDim.x + threadIdx.x; C < NC; C += gridDim.x * blockDim.x) {
        const int X = C % A.mx, Y = C / A.mx;
        unsigned long long msk = 0;
        for (int l = 0; l < A.m * A.m; ++l) {          // P5 spins of the subarray's cells
            const uint32_t c = (uint32_t)(Y * A.m + l / A.m) * (uint32_t)A.nx + (uint32_t)(X * A.m + l % A.m);
            const u32x4 r = philox4x32_10_rk(0u, c, 0u, 1u, A.rk);
            if ((unsigned long long)r.x >= A.thr_init) msk |= 1ull << l;
        }
        const u32x4 r = philox4x32_10_rk(0u, (uint32_t)C, 0u, A.tag_i, A.rk);
        uint64_t q = nlog_q32(((uint64_t)r.y << 32) | r.z, lr, ACA_LN2_Q48);
        q = (__umul64hi(q, A.inv) << 32) | ((q * A.inv) >> 32);
        A.mask[C] = msk;
        A.T[C] = q < 1 ? 1 : q;
        A.n[C] = 0u;
    }
}

__device__ __forceinline__ bool agg_below(unsigned long long t, int C, unsigned long long t2, int C2) {
    return t < t2 || (t == t2 && C < C2);
}

__global__ void __launch_bounds__(256) agg_round_kernel(const AggParams A, const unsigned long long* __restrict__ lr_g,
                                                        AggAcc* __restrict__ acc) {
    __shared__ unsigned long long lr[512];
    __shared__ unsigned long long red[5][8];
    for (int i = threadIdx.x; i < 512; i += blockDim.x) lr[i] = lr_g[i];
    __syncthreads();
    const int NC = A.mx * A.my;
    const int m = A.m;
    volatile unsigned long long* VT = A.T;
    volatile unsigned long long* VM = A.mask;
    unsigned long long arr = 0, flips = 0, hsh = 0, active = 0, blocked = 0;
    for (int C = blockIdx.x * blockDim.x + threadIdx.x; C < NC; C += gridDim.x * blockDim.x) {
        const int X = C % A.mx, Y = C / A.mx;
        const int Cl = Y * A.mx + (X == 0 ? A.mx - 1 : X - 1), Cr = Y * A.mx + (X == A.mx - 1 ? 0 : X + 1);
        const int Cu = (Y == 0 ? A.my - 1 : Y - 1) * A.mx + X, Cd = (Y == A.my - 1 ? 0 : Y + 1) * A.mx + X;
        unsigned long long T = A.T[C], msk = A.mask[C];
        unsigned int k = A.n[C];
        int b = 0;
        for (; b < A.budget && T < A.Tend; ++b) {
            const u32x4 r = philox4x32_10_rk(k, (uint32_t)C, 0u, A.tag_e, A.rk);
            const int l = A.lg == 0 ? 0 : (int)(r.w >> (32 - A.lg));
            const int i = l % m, j = l / m;
            // Step 3: wait for the subarrays holding the cell's outside neighbours (W(c))
            bool ok = true;
            unsigned long long ml = 0, mr = 0, mu = 0, md = 0;
            if (i == 0 && Cl != C) { ok = ok && agg_below(T, C, VT[Cl], Cl); }
            if (i == m - 1 && Cr != C) { ok = ok && agg_below(T, C, VT[Cr], Cr); }
            if (j == 0 && Cu != C) { ok = ok && agg_below(T, C, VT[Cu], Cu); }
            if (j == m - 1 && Cd != C) { ok = ok && agg_below(T, C, VT[Cd], Cd); }
            if (!ok) { ++blocked; break; }
            __threadfence();                       // acquire: masks after the times we checked
            if (i == 0) ml = Cl == C ? msk : VM[Cl];
            if (i == m - 1) mr = Cr == C ? msk : VM[Cr];
            if (j == 0) mu = Cu == C ? msk : VM[Cu];
            if (j == m - 1) md = Cd == C ? msk : VM[Cd];
            // Step 4: neighbour spins (+1 bits), periodic within the torus
            const uint32_t left = i > 0 ? (uint32_t)(msk >> (l - 1)) & 1u : (uint32_t)(ml >> (j * m + m - 1)) & 1u;
            const uint32_t right = i < m - 1 ? (uint32_t)(msk >> (l + 1)) & 1u : (uint32_t)(mr >> (j * m)) & 1u;
            const uint32_t up = j > 0 ? (uint32_t)(msk >> (l - m)) & 1u : (uint32_t)(mu >> ((m - 1) * m + i)) & 1u;
            const uint32_t down = j < m - 1 ? (uint32_t)(msk >> (l + m)) & 1u : (uint32_t)(md >> i) & 1u;
            const uint32_t sb = (uint32_t)(msk >> l) & 1u;
            const uint32_t idx = (left + right + up + down) + 5u * sb;
            const uint32_t flip = (unsigned long long)r.x < A.thr[idx] ? 1u : 0u;
            uint64_t q = nlog_q32(((uint64_t)r.y << 32) | r.z, lr, ACA_LN2_Q48);
            q = (__umul64hi(q, A.inv) << 32) | ((q * A.inv) >> 32);
            q = q < 1 ? 1 : q;
            if (A.do_hash)
                hsh += ev_hash(r.w, T, ((unsigned long long)l << 1) ^ (unsigned long long)(sb ^ flip));
            msk ^= (unsigned long long)flip << l;
            flips += flip;
            ++arr;
            ++k;
            T += q;
            // publish: mask, fence, time (release)
            VM[C] = msk;
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
// Kernel classes of an m x m subarray (bit l = j m + i of the spin mask S): the number of +1
// neighbours of every kernel cell by bit-sliced adders over the four shifted masks (kernel
// neighbours are inside the subarray), then the ten class masks M[idx(s, Sigma)], idx = ones +
// 5 s (P4). Returns W = |Gamma_0| 2^32 + sum_k popc(M_k) thr_k.
__device__ __forceinline__ unsigned long long bkl_classes(unsigned long long S, int m, unsigned long long K,
                                                          const unsigned long long* thr, unsigned long long* M,
                                                          unsigned long long W0) {
    const unsigned long long L = S << 1, R = S >> 1, U = S << m, D = S >> m;
    const unsigned long long h1 = L ^ R, k1 = L & R, h2 = U ^ D, k2 = U & D;
    const unsigned long long p0 = h1 ^ h2, c = h1 & h2;
    const unsigned long long q0 = k1 ^ k2 ^ c, q1 = (k1 & k2) | (c & (k1 ^ k2));   // ones = p0 + 2 q0 + 4 q1
    unsigned long long W = W0;
#pragma unroll
    for (int j = 0; j <= 4; ++j) {
        const unsigned long long e = ((j & 1) ? p0 : ~p0) & ((j & 2) ? q0 : ~q0) & ((j & 4) ? q1 : ~q1) & K;
        M[j] = e & ~S;           // s = -1
        M[j + 5] = e & S;        // s = +1
        W += (unsigned long long)__popcll(M[j]) * thr[j] + (unsigned long long)__popcll(M[j + 5]) * thr[j + 5];
    }
    return W;
}

// index of the r-th set bit (r = 0, 1, ...) of a 64-bit mask
__device__ __forceinline__ int nth_set_bit(unsigned long long x, unsigned int r) {
    const unsigned int lo = (unsigned int)x, plo = __popc(lo);
    if (r < plo) return (int)__fns(lo, 0, (int)r + 1);
    return 32 + (int)__fns((unsigned int)(x >> 32), 0, (int)(r - plo) + 1);
}

__device__ __forceinline__ unsigned long long bkl_inv(double lambda, unsigned long long W) {
    return (unsigned long long)floor(18446744073709551616.0 / (lambda * (double)W) + 0.5);
}

struct BklExtra {
    double lambda;
    unsigned long long K, B;      // kernel and boundary-layer masks of a subarray
    unsigned long long W0;        // |Gamma_0| 2^32
};

__global__ void bkl_init_kernel(const AggParams A, const BklExtra E, const unsigned long long* __restrict__ lr_g) {
    __shared__ unsigned long long lr[512];
    for (int i = threadIdx.x; i < 512; i += blockDim.x) lr[i] = lr_g[i];
    __syncthreads();
    const int NC = A.mx * A.my;
    for (int C = blockIdx.x * blockDim.x + threadIdx.x; C < NC; C += gridDim.x * blockDim.x) {
        const int X = C % A.mx, Y = C / A.mx;
        unsigned long long msk = 0;
        for (int l = 0; l < A.m * A.m; ++l) {
            const uint32_t c = (uint32_t)(Y * A.m + l / A.m) * (uint32_t)A.nx + (uint32_t)(X * A.m + l % A.m);
            const u32x4 r = philox4x32_10_rk(0u, c, 0u, 1u, A.rk);
            if ((unsigned long long)r.x >= A.thr_init) msk |= 1ull << l;
        }
        unsigned long long M[10];
        const unsigned long long W = bkl_classes(msk, A.m, E.K, A.thr, M, E.W0);
        const u32x4 r = philox4x32_10_rk(0u, (uint32_t)C, 0u, 6u, A.rk);
        const uint64_t q = nlog_q32(((uint64_t)r.z << 32) | r.w, lr, ACA_LN2_Q48);
        const unsigned long long inv = bkl_inv(E.lambda, W);
        const uint64_t d = (__umul64hi(q, inv) << 32) | ((q * inv) >> 32);
        A.mask[C] = msk;
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
    volatile unsigned long long* VM = A.mask;
    unsigned long long arr = 0, flips = 0, hsh = 0, active = 0, blocked = 0;
    for (int C = blockIdx.x * blockDim.x + threadIdx.x; C < NC; C += gridDim.x * blockDim.x) {
        const int X = C % A.mx, Y = C / A.mx;
        const int Cl = Y * A.mx + (X == 0 ? A.mx - 1 : X - 1), Cr = Y * A.mx + (X == A.mx - 1 ? 0 : X + 1);
        const int Cu = (Y == 0 ? A.my - 1 : Y - 1) * A.mx + X, Cd = (Y == A.my - 1 ? 0 : Y + 1) * A.mx + X;
        unsigned long long T = A.T[C], msk = A.mask[C];
        unsigned int k = A.n[C];
        for (int b = 0; b < A.budget && T < A.Tend; ++b) {
            const u32x4 r = philox4x32_10_rk(k, (uint32_t)C, 0u, 5u, A.rk);
            unsigned long long M[10];
            const unsigned long long W = bkl_classes(msk, m, E.K, A.thr, M, E.W0);
            const unsigned long long Xr = ((unsigned long long)r.x << 32) | r.y;
            const unsigned long long u = __umul64hi(Xr, W);
            int l;
            uint32_t sb, flip;
            if (u < E.W0) {   // boundary layer: the standard model, after waiting for W(c)
                l = nth_set_bit(E.B, (unsigned int)(u >> 32));
                const int i = l % m, j = l / m;
                bool ok = true;
                if (i == 0 && Cl != C) ok = ok && agg_below(T, C, VT[Cl], Cl);
                if (i == m - 1 && Cr != C) ok = ok && agg_below(T, C, VT[Cr], Cr);
                if (j == 0 && Cu != C) ok = ok && agg_below(T, C, VT[Cu], Cu);
                if (j == m - 1 && Cd != C) ok = ok && agg_below(T, C, VT[Cd], Cd);
                if (!ok) { ++blocked; break; }
                __threadfence();
                unsigned long long ml = 0, mr = 0, mu = 0, md = 0;
                if (i == 0) ml = Cl == C ? msk : VM[Cl];
                if (i == m - 1) mr = Cr == C ? msk : VM[Cr];
                if (j == 0) mu = Cu == C ? msk : VM[Cu];
                if (j == m - 1) md = Cd == C ? msk : VM[Cd];
                const uint32_t left = i > 0 ? (uint32_t)(msk >> (l - 1)) & 1u : (uint32_t)(ml >> (j * m + m - 1)) & 1u;
                const uint32_t right = i < m - 1 ? (uint32_t)(msk >> (l + 1)) & 1u : (uint32_t)(mr >> (j * m)) & 1u;
                const uint32_t up = j > 0 ? (uint32_t)(msk >> (l - m)) & 1u : (uint32_t)(mu >> ((m - 1) * m + i)) & 1u;
                const uint32_t down = j < m - 1 ? (uint32_t)(msk >> (l + m)) & 1u : (uint32_t)(md >> i) & 1u;
                sb = (uint32_t)(msk >> l) & 1u;
                flip = (unsigned long long)(u & 0xffffffffull) < A.thr[(left + right + up + down) + 5u * sb] ? 1u : 0u;
            } else {          // kernel: pick the class, then its cell; the cell flips
                unsigned long long o = u - E.W0;
                int kc = 0;
#pragma unroll
                for (int q = 0; q < 9; ++q) {
                    const unsigned long long Wk = (unsigned long long)__popcll(M[kc]) * A.thr[kc];
                    if (o < Wk) break;
                    o -= Wk;
                    ++kc;
                }
                l = nth_set_bit(M[kc], (unsigned int)(o / A.thr[kc]));
                sb = (uint32_t)(msk >> l) & 1u;
                flip = 1u;
            }
            if (A.do_hash)
                hsh += ev_hash(r.w, T, ((unsigned long long)l << 1) ^ (unsigned long long)(sb ^ flip));
            msk ^= (unsigned long long)flip << l;
            flips += flip;
            ++arr;
            ++k;
            unsigned long long M2[10];
            const unsigned long long W2 = bkl_classes(msk, m, E.K, A.thr, M2, E.W0);
            const uint64_t q = nlog_q32(((uint64_t)r.z << 32) | r.w, lr, ACA_LN2_Q48);
            const unsigned long long inv = bkl_inv(E.lambda, W2);
            const uint64_t d = (__umul64hi(q, inv) << 32) | ((q * inv) >> 32);
            T += d < 1 ? 1 : d;
            VM[C] = msk;
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

// Spins of the torus (int8, row-major) from the masks.
__global__ void agg_unpack_kernel(const AggParams A, int8_t* __restrict__ spins) {
    const long long N = (long long)A.nx * A.ny;
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < N; c += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(c % A.nx), y = (int)(c / A.nx);
        const int C = (y / A.m) * A.mx + x / A.m, l = (y % A.m) * A.m + x % A.m;
        spins[c] = (A.mask[C] >> l) & 1ull ? (int8_t)1 : (int8_t)-1;
    }
}

}  // namespace aca
