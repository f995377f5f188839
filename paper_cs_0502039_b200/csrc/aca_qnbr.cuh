// aca_qnbr.cuh — the Ising model on the q-th degree neighbourhood (Eq. nei2 / neiq,
// PAPER.md:991-1030; docs/PRIMITIVES.md P12) on the GPU.
//
// neighbors^q(c) is the L1 ball of radius q around c (|neighbors^q| - 1 = 2q(q+1) in 2-D): a cell
// fires only when its (t, c) is below that of every member, and its flip uses the spin sum over
// all of them. "It is easy to rewrite the algorithms ... for the case q > 1":
// here fig:s1c1pe's synchronous rounds run inside a CTA on a tile staged in shared memory with a
// halo of width q (the frozen W(c) layer of PAPER.md:741-750). With q >= 2 the neighbourhood has
// diagonal members, so the checkerboard of the one-cell path is not enough: tiles are coloured
// per axis (0/1 alternating, 2 for the last tile of an odd count) and one launch runs the tiles of
// one colour; two tiles of a colour are at least one tile (>= q cells) apart along some axis, so no
// tile modifies a cell another tile of the launch reads. A tile visit: stage the tile and its halo
// (times, spins) and the counters of its cells; rounds of (test all own cells against their
// members -> draw and compute privately -> barrier -> commit -> barrier) until a round fires
// nothing or R rounds; write back. Every fired cell is a strict (t, c) minimum of its
// neighbourhood with exact values, so the trajectory is the serial one.
#pragma once
#include "aca_kernels.cuh"

namespace aca {

constexpr int QN_MAXZ = 128;          // 3-D, q = 4
constexpr int QN_THREADS = 256;

struct QParams {
    unsigned long long* t;            // [N] pending arrival times, Q32
    signed char* s;                   // [N] spins +-1
    unsigned int* n;                  // [N] arrival counters
    int ndim, q, nofs;
    int dim[3];                       // nx, ny, nz (1 for 2-D)
    int ntl[3];                       // tiles per axis (>= 2 each used axis)
    int ncol[3];                      // colours per axis: 2, or 3 for an odd tile count
    int tmax[3];                      // largest tile extent per axis
    int colour;                       // this launch: cx + ncol0 (cy + ncol1 cz)
    int R;                            // rounds per tile visit
    int tie_bits, law;
    uint32_t rk[20];
    unsigned long long inv, Tend, thr_init;
    const int* ofs;                   // [nofs][3]
    const unsigned long long* thr;    // [2 (nofs + 1)] P4 table
};

struct QAcc {
    unsigned long long arrivals, flips, hash, active;
    long long B2, M;
};

__device__ __forceinline__ int qn_tile_lo(int k, int d, int nt) { return (int)(((long long)k * d) / nt); }

__global__ void qn_init_kernel(const QParams P, const unsigned long long* __restrict__ lr_g) {
    __shared__ unsigned long long lr[512];
    for (int i = threadIdx.x; i < 512; i += blockDim.x) lr[i] = lr_g[i];
    __syncthreads();
    const long long N = (long long)P.dim[0] * P.dim[1] * P.dim[2];
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < N; c += (long long)gridDim.x * blockDim.x) {
        const u32x4 r = philox4x32_10_rk(0u, (uint32_t)c, (uint32_t)(c >> 32), 1u, P.rk);   // P5
        P.s[c] = (unsigned long long)r.x < P.thr_init ? (signed char)-1 : (signed char)1;
        P.t[c] = delta_q32(r.y, r.z, lr, ACA_LN2_Q48, P.inv, P.tie_bits, P.law);
        P.n[c] = 0u;
    }
}

// One tile visit per CTA for the tiles of colour P.colour.
__global__ void __launch_bounds__(QN_THREADS) qn_tile_kernel(const QParams P, const unsigned long long* __restrict__ lr_g,
                                                              QAcc* __restrict__ acc) {
    extern __shared__ __align__(16) unsigned char qsm[];
    __shared__ unsigned long long lr[512];
    __shared__ unsigned long long thr[2 * (QN_MAXZ + 1)];
    __shared__ int dofs[QN_MAXZ];
    __shared__ unsigned long long red[4][QN_THREADS / 32];
    const int q = P.q, nofs = P.nofs;
    // this CTA's tile: decompose blockIdx over the tiles of the colour
    int cx = P.colour % P.ncol[0], cy = (P.colour / P.ncol[0]) % P.ncol[1], cz = P.colour / (P.ncol[0] * P.ncol[1]);
    int cc[3] = {cx, cy, cz}, cnt[3], k[3];
    for (int a = 0; a < 3; ++a) {   // tiles of colour c along axis a: c, c + 2, ... (colour 2: the last one)
        const int nt = P.ntl[a];
        if (a >= P.ndim) { cnt[a] = 1; continue; }
        if (cc[a] == 2) cnt[a] = 1;
        else cnt[a] = (P.ncol[a] == 3 ? nt - 1 - cc[a] + 1 : nt - cc[a] + 1) / 2;
    }
    int b = blockIdx.x;
    for (int a = 0; a < 3; ++a) {
        const int j = b % cnt[a];
        b /= cnt[a];
        k[a] = a >= P.ndim ? 0 : (cc[a] == 2 ? P.ntl[a] - 1 : cc[a] + 2 * j);
    }
    int lo[3], ex[3], SX[3];
    for (int a = 0; a < 3; ++a) {
        if (a >= P.ndim) { lo[a] = 0; ex[a] = 1; SX[a] = 1; continue; }
        lo[a] = qn_tile_lo(k[a], P.dim[a], P.ntl[a]);
        ex[a] = qn_tile_lo(k[a] + 1, P.dim[a], P.ntl[a]) - lo[a];
        SX[a] = P.tmax[a] + 2 * q;
    }
    const int hz = P.ndim == 3 ? q : 0;
    const int RX = ex[0] + 2 * q, RY = ex[1] + 2 * q, RZ = ex[2] + 2 * hz;
    const int SXY = SX[0] * SX[1];
    const int nreg = SXY * (P.ndim == 3 ? SX[2] : 1);
    const int ni = ex[0] * ex[1] * ex[2];
    const int nimax = P.tmax[0] * P.tmax[1] * (P.ndim == 3 ? P.tmax[2] : 1);
    unsigned long long* Ts = (unsigned long long*)qsm;                 // [nreg]
    unsigned long long* Tn = Ts + nreg;                                // [nimax] pending new time (0: none)
    unsigned int* Ns = (unsigned int*)(Tn + nimax);                    // [nimax]
    signed char* Ss = (signed char*)(Ns + nimax);                      // [nreg]
    signed char* Sn = Ss + nreg;                                       // [nimax]
    for (int i = threadIdx.x; i < 512; i += blockDim.x) lr[i] = lr_g[i];
    for (int i = threadIdx.x; i < 2 * (nofs + 1); i += blockDim.x) thr[i] = P.thr[i];
    for (int j = threadIdx.x; j < nofs; j += blockDim.x)
        dofs[j] = P.ofs[3 * j] + SX[0] * P.ofs[3 * j + 1] + SXY * P.ofs[3 * j + 2];
    // stage the region [lo - q, lo + ex + q) per axis (wrapped), and the own counters
    const int nx = P.dim[0], ny = P.dim[1], nz = P.dim[2];
    for (int r = threadIdx.x; r < RX * RY * RZ; r += blockDim.x) {
        const int rx = r % RX, ry = (r / RX) % RY, rz = r / (RX * RY);
        const int gx = (lo[0] - q + rx + q * nx) % nx, gy = (lo[1] - q + ry + q * ny) % ny;
        const int gz = (lo[2] - hz + rz + hz * nz) % nz;
        const long long g = ((long long)gz * ny + gy) * nx + gx;
        const int ri = rx + SX[0] * ry + SXY * rz;
        Ts[ri] = P.t[g];
        Ss[ri] = P.s[g];
    }
    for (int i = threadIdx.x; i < ni; i += blockDim.x) {
        const int x = i % ex[0], y = (i / ex[0]) % ex[1], z = i / (ex[0] * ex[1]);
        Ns[i] = P.n[((long long)(lo[2] + z) * ny + lo[1] + y) * nx + lo[0] + x];
        Tn[i] = 0ull;
    }
    __syncthreads();
    unsigned long long arr = 0, flips = 0, hsh = 0;
    const int z2 = nofs;
    for (int round = 0; round < P.R; ++round) {
        int fired = 0;
        for (int i = threadIdx.x; i < ni; i += blockDim.x) {
            const int x = i % ex[0], y = (i / ex[0]) % ex[1], z = i / (ex[0] * ex[1]);
            const int ri = (x + q) + SX[0] * (y + q) + SXY * (z + hz);
            const unsigned long long t = Ts[ri];
            if (t >= P.Tend) continue;
            const long long c = ((long long)(lo[2] + z) * ny + lo[1] + y) * nx + lo[0] + x;
            bool ok = true;
            int sig = 0;
            for (int j = 0; j < nofs && ok; ++j) {
                const int rj = ri + dofs[j];
                const unsigned long long t2 = Ts[rj];
                if (t2 < t) ok = false;
                else if (t2 == t) {   // tie: (t, c) order on the global ids (P6)
                    const int rx = rj % SX[0], ry = (rj / SX[0]) % SX[1], rz = rj / SXY;
                    const int gx = (lo[0] - q + rx + q * nx) % nx, gy = (lo[1] - q + ry + q * ny) % ny;
                    const int gz = (lo[2] - hz + rz + hz * nz) % nz;
                    if (((long long)gz * ny + gy) * nx + gx < c) ok = false;
                }
                sig += Ss[rj];
            }
            if (!ok) continue;
            const int sc = Ss[ri];
            const u32x4 r = philox4x32_10_rk(Ns[i], (uint32_t)c, (uint32_t)((unsigned long long)c >> 32), 0u, P.rk);
            const int idx = (sig + z2) / 2 + (z2 + 1) * (sc + 1) / 2;
            const int ns = (unsigned long long)r.x < thr[idx] ? -sc : sc;
            flips += ns != sc;
            arr += 1;
            hsh += ev_hash(r.w, t, ns > 0 ? 1ull : 0ull);
            Tn[i] = t + delta_q32(r.y, r.z, lr, ACA_LN2_Q48, P.inv, P.tie_bits, P.law);
            Sn[i] = (signed char)ns;
            fired = 1;
        }
        if (!__syncthreads_or(fired)) break;
        for (int i = threadIdx.x; i < ni; i += blockDim.x) {   // commit (fig:s1c1pe steps 6-7)
            const unsigned long long tn = Tn[i];
            if (!tn) continue;
            const int x = i % ex[0], y = (i / ex[0]) % ex[1], z = i / (ex[0] * ex[1]);
            const int ri = (x + q) + SX[0] * (y + q) + SXY * (z + hz);
            Ts[ri] = tn;
            Ss[ri] = Sn[i];
            Ns[i] += 1u;
            Tn[i] = 0ull;
        }
        __syncthreads();
    }
    unsigned long long active = 0;
    for (int i = threadIdx.x; i < ni; i += blockDim.x) {   // write back the own cells
        const int x = i % ex[0], y = (i / ex[0]) % ex[1], z = i / (ex[0] * ex[1]);
        const int ri = (x + q) + SX[0] * (y + q) + SXY * (z + hz);
        const long long g = ((long long)(lo[2] + z) * ny + lo[1] + y) * nx + lo[0] + x;
        P.t[g] = Ts[ri];
        P.s[g] = Ss[ri];
        P.n[g] = Ns[i];
        active += Ts[ri] < P.Tend;
    }
    unsigned long long v[4] = {arr, flips, hsh, active};
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int a = 0; a < 4; ++a) {
        unsigned long long x = v[a];
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (!lane) red[a][w] = x;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        unsigned long long x = 0;
        for (int j = 0; j < QN_THREADS / 32; ++j) x += red[threadIdx.x][j];
        if (x) atomicAdd(&acc->arrivals + threadIdx.x, x);
    }
}

// B2 = sum_c s(c) sum_{c' in neighbors^q(c) \ {c}} s(c') (= 2 B) and M.
__global__ void qn_stats_kernel(const QParams P, QAcc* __restrict__ acc) {
    __shared__ long long red[2][QN_THREADS / 32];
    const int nx = P.dim[0], ny = P.dim[1], nz = P.dim[2], q = P.q;
    const long long N = (long long)nx * ny * nz;
    long long b2 = 0, m = 0;
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < N; c += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(c % nx), y = (int)((c / nx) % ny), z = (int)(c / ((long long)nx * ny));
        int sig = 0;
        for (int j = 0; j < P.nofs; ++j) {
            const int gx = (x + P.ofs[3 * j] + q * nx) % nx, gy = (y + P.ofs[3 * j + 1] + q * ny) % ny;
            const int gz = (z + P.ofs[3 * j + 2] + q * nz) % nz;
            sig += P.s[((long long)gz * ny + gy) * nx + gx];
        }
        b2 += (long long)P.s[c] * sig;
        m += P.s[c];
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 16; o; o >>= 1) {
        b2 += __shfl_xor_sync(0xffffffffu, b2, o);
        m += __shfl_xor_sync(0xffffffffu, m, o);
    }
    if (!lane) { red[0][w] = b2; red[1][w] = m; }
    __syncthreads();
    if (threadIdx.x < 2) {
        long long x = 0;
        for (int j = 0; j < QN_THREADS / 32; ++j) x += red[threadIdx.x][j];
        atomicAdd((unsigned long long*)(&acc->B2 + threadIdx.x), (unsigned long long)x);
    }
}

}  // namespace aca
