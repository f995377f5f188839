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
                hsh += mix64(T ^ rotl64((unsigned long long)C, 20) ^ rotl64((unsigned long long)k, 44) ^
                             ((unsigned long long)l << 1) ^ (unsigned long long)(sb ^ flip));
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
