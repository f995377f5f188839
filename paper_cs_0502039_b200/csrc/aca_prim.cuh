// aca_prim.cuh — device primitives of the method, implemented from docs/PRIMITIVES.md.
// Shares no code with oracle/ (which implements the same text in plain C).
#pragma once
#include <stdint.h>

#include "gauss_tables.cuh"

namespace aca {

// ---------------------------------------------------------------- P1 Philox4x32-10
// Counter-based per-cell stream: condition (i) of PAPER.md:581-582 ("for the same cell,
// the pseudo-random sequence is always the same"), r(n) of Eq. newt1i.
struct u32x4 { uint32_t x, y, z, w; };

__device__ __forceinline__ u32x4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;   // IMAD.WIDE.U32
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        c1 = (uint32_t)p1;
        c3 = (uint32_t)p0;
        c0 = n0;
        c2 = n2;
        if (r < 9) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    }
    return {c0, c1, c2, c3};
}

// Same function with the ten round keys precomputed (rk[2r], rk[2r+1] = key schedule of round
// r, see philox_round_keys). With rk in the kernel-parameter (constant) bank the key xor folds
// into the LOP3 of each round: 2 IMAD.WIDE + 2 LOP3 per round.
__device__ __forceinline__ u32x4 philox4x32_10_rk(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                   const uint32_t* rk) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ rk[2 * r];
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ rk[2 * r + 1];
        c1 = (uint32_t)p1;
        c3 = (uint32_t)p0;
        c0 = n0;
        c2 = n2;
    }
    return {c0, c1, c2, c3};
}

__host__ __device__ inline void philox_round_keys(uint32_t k0, uint32_t k1, uint32_t* rk) {
    for (int r = 0; r < 10; ++r) {
        rk[2 * r] = k0;
        rk[2 * r + 1] = k1;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

// ---------------------------------------------------------------- P3 NLOG-2
// Table views. NLOG-2 reads L[i] (u64) and the low word of R[i] (R[0] = 2^32 is handled by the
// i = 0 case). NlogLR: the interleaved {L[i], R[i]} u64 pairs of ACA_NLOG_LR (global or shared
// memory, generic addressing). NlogSmem: the two tables split in shared memory (L u64[256],
// R u32[256]) and addressed by 32-bit shared-window offsets: a warp's 32 random lookups then
// spread over 16 (L) and 32 (R) bank groups instead of the 8 of the 16-byte interleaved
// entries, and no generic-to-shared address conversion is repeated per lookup.
struct NlogLR {
    const unsigned long long* lr;
    __device__ __forceinline__ uint64_t L(uint32_t i) const { return lr[2 * i]; }
    __device__ __forceinline__ uint32_t R(uint32_t i) const { return (uint32_t)lr[2 * i + 1]; }
};
struct NlogSmem {
    uint32_t l, r;   // shared-window byte offsets of L[0] and R[0]
    __device__ __forceinline__ uint64_t L(uint32_t i) const {
        uint64_t v;
        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(l + 8u * i));
        return v;
    }
    __device__ __forceinline__ uint32_t R(uint32_t i) const {
        uint32_t v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(r + 4u * i));
        return v;
    }
};

// -ln(u) in Q32 for u = (X|1)/2^64, integer-only (docs/PRIMITIVES.md P3). Every intermediate
// of the definition fits 32 bits except L + A, so the arithmetic is done on 32-bit halves
// (IMAD / IMAD.HI) — the same integers as the 64-bit statement of P3:
//   V = (g R[i]) >> 32 = umulhi(g, R[i] mod 2^32) + [i = 0] g     (R[0] = 2^32, R[i>0] < 2^32)
//   V2 = V^2 = (v2h, v2l);  B = ceil(V2 / 2^33);  C = floor((umulhi(v2h, V) >> 8) / 3)
//   Wq = ceil(V2 / 2^32) < 2^32;  D = ceil(Wq^2 / 2^50)
//   lnf = L[i] + (V << 8) + C - (B + D)   (B + D < 2^32; the sum is exact modulo 2^64)
template <class Tab>
__device__ __forceinline__ uint64_t nlog_q32_t(uint64_t X, const Tab& tab, uint64_t ln2_q48) {
    const uint64_t x = X | 1ull;
    const uint32_t xh = (uint32_t)(x >> 32), xl = (uint32_t)x;
    int z;
    uint32_t mh, ml;   // m = x << (z + 1) mod 2^64, the mantissa bits below the leading one
    if (xh != 0u) {    // all but 2^-32 of the draws: 32-bit leading-zero count and funnel shifts
        z = __clz((int)xh);
        mh = __funnelshift_lc(xl, xh, z + 1);
        ml = __funnelshift_lc(0u, xl, z + 1);
    } else {
        z = __clzll((long long)x);
        const uint64_t m = (x << z) << 1;
        mh = (uint32_t)(m >> 32);
        ml = (uint32_t)m;
    }
    const uint32_t i = mh >> 24;
    const uint32_t g = __funnelshift_r(ml, mh, 24);          // bits 24..55 of m
    const uint64_t Li = tab.L(i);
    const uint32_t V = i == 0u ? g : __umulhi(g, tab.R(i));
    const uint32_t v2l = V * V, v2h = __umulhi(V, V);
    const uint32_t B = (v2h >> 1) + ((v2l | (v2h & 1u)) != 0u ? 1u : 0u);
    const uint32_t C = (__umulhi(v2h, V) >> 8) / 3u;
    const uint32_t Wq = v2h + (v2l != 0u ? 1u : 0u);
    const uint32_t w2l = Wq * Wq, w2h = __umulhi(Wq, Wq);
    const uint32_t D = (w2h >> 18) + ((w2l | (w2h & 0x3ffffu)) != 0u ? 1u : 0u);
    const uint64_t lnf = Li + ((uint64_t)V << 8) + (uint64_t)C - (uint64_t)(B + D);
    const uint64_t S = (uint64_t)(uint32_t)(z + 1) * ln2_q48 - lnf;
    return (S + (1ull << 15)) >> 16;
}
__device__ __forceinline__ uint64_t nlog_q32(uint64_t X, const unsigned long long* __restrict__ lr,
                                             uint64_t ln2_q48) {
    return nlog_q32_t(X, NlogLR{lr}, ln2_q48);
}

// The standard normal quantile z = Phi^{-1}((w + 1/2) 2^-32) of P3L laws 3 and 4 (docs/PRIMITIVES.md
// P3L): by symmetry on p' = min(p, 1 - p), s = sqrt(-ln p') with -ln p' from NLOG-2 (exact integers),
// |z| = G(s) by the cubic pieces of ACA_GAUSS_C (Horner in IEEE double through the _rn intrinsics,
// which are never contracted into FMAs: the same roundings as the oracle's plain C).
template <class Tab>
__device__ __forceinline__ double gauss_z(uint32_t w, const Tab& tab, uint64_t ln2_q48) {
    const uint32_t wp = w < 0x80000000u ? w : 0xffffffffu - w;
    const uint64_t q = nlog_q32_t(((uint64_t)(2ull * wp + 1ull)) << 31, tab, ln2_q48);
    const double s = __dsqrt_rn(__dmul_rn((double)q, 1.0 / 4294967296.0));
    const double u = __dmul_rn(__dadd_rn(s, -0.828125), 256.0);
    int i = (int)u;
    i = i < 0 ? 0 : (i > 1023 ? 1023 : i);
    const double t = __dadd_rn(u, -(double)i);
    const double* c = ACA_GAUSS_C + 4 * i;
    const double g = __dadd_rn(__dmul_rn(__dadd_rn(__dmul_rn(__dadd_rn(__dmul_rn(c[3], t), c[2]), t), c[1]), t), c[0]);
    return w < 0x80000000u ? -g : g;
}
// A Gaussian period of mean 1 and sd 1/4 in Q32, U = floor((1 + z/4) 2^32); a period below one unit
// is redrawn from the sub-draws a0 of Philox ctr (sa, sb, j, tag), j = 1..31, under the fixed key
// (0x243F6A88, 0x85A308D3); U = 1 if all 32 draws fail.
template <class Tab>
__device__ __forceinline__ uint64_t gauss_u(uint32_t w, uint32_t sa, uint32_t sb, uint32_t tag, const Tab& tab,
                                            uint64_t ln2_q48) {
    for (uint32_t j = 0;; ++j) {
        const double x = __dmul_rn(__dadd_rn(1.0, __dmul_rn(0.25, gauss_z(w, tab, ln2_q48))), 4294967296.0);
        if (x >= 1.0) return (uint64_t)floor(x);
        if (j == 31) return 1ull;
        w = philox4x32_10(sa, sb, j + 1u, tag, 0x243F6A88u, 0x85A308D3u).x;
    }
}

// P3L asynchrony law: the unscaled increment U in Q32 (docs/PRIMITIVES.md P3L).
//   0 Poisson, Eq. newt1i:   U = NLOG-2((w1 << 32) | w2)
//   1 uniform on (0,1):    U = w1
//   2 r^(1/8):             U = floor(sqrt(sqrt(sqrt(r))) * 2^32), r = (w1 + 0.5) 2^-32
//     (IEEE double; sqrt is correctly rounded on the device as on the host)
//   3 Gaussian period (the liberal reading): U = gauss_u(w1, w1, w2, 9), a fresh
//     period of mean 1/lambda and sd 1/(4 lambda) at every arrival
//   4 (the strict reading) needs the cell: cell_period_q32
template <class Tab>
__device__ __forceinline__ uint64_t law_q32_t(uint32_t w1, uint32_t w2, const Tab& tab, uint64_t ln2_q48, int law) {
    if (law == 1) return (uint64_t)w1;
    if (law == 3) return gauss_u(w1, w1, w2, 9u, tab, ln2_q48);
    if (law == 2) {
        const double r = ((double)w1 + 0.5) * (1.0 / 4294967296.0);
        return (uint64_t)(__dsqrt_rn(__dsqrt_rn(__dsqrt_rn(r))) * 4294967296.0);
    }
    return nlog_q32_t(((uint64_t)w1 << 32) | w2, tab, ln2_q48);
}
__device__ __forceinline__ uint64_t law_q32(uint32_t w1, uint32_t w2, const unsigned long long* lr, uint64_t ln2_q48,
                                            int law) {
    return law_q32_t(w1, w2, NlogLR{lr}, ln2_q48, law);
}

// Law 4, the strict reading of PAPER.md:404-410 (sigma_c = 0, m_c itself Gaussian): the fixed period
// of cell c from the spare word w3 of its initial draw (Philox ctr (0, c_lo, c_hi, 1), run key).
template <class Tab>
__device__ __forceinline__ uint64_t cell_period_q32(uint32_t c_lo, uint32_t c_hi, const uint32_t* rk, const Tab& tab,
                                                    uint64_t ln2_q48) {
    const u32x4 r = philox4x32_10_rk(0u, c_lo, c_hi, 1u, rk);
    return gauss_u(r.w, r.w, c_lo, 10u, tab, ln2_q48);
}

// Delta = max(1, (U INV) >> 32) and the P3b tie quantisation.
__device__ __forceinline__ uint64_t delta_of_u(uint64_t q, uint64_t inv_lambda, int tie_bits) {
    uint64_t d;
    if (inv_lambda == (1ull << 32)) {
        d = q;
    } else {
        d = (__umul64hi(q, inv_lambda) << 32) | ((q * inv_lambda) >> 32);
    }
    d = d < 1ull ? 1ull : d;
    if (tie_bits > 0) {
        const uint64_t quantum = 1ull << tie_bits;
        d &= ~(quantum - 1ull);
        d = d < quantum ? quantum : d;
    }
    return d;
}

// next_t = t + U / lambda, next_t > t.
template <class Tab>
__device__ __forceinline__ uint64_t delta_q32_t(uint32_t w1, uint32_t w2, const Tab& tab, uint64_t ln2_q48,
                                                uint64_t inv_lambda, int tie_bits, int law = 0) {
    return delta_of_u(law_q32_t(w1, w2, tab, ln2_q48, law), inv_lambda, tie_bits);
}
// The increment of cell c at any arrival: law 4 the cell's fixed period, every other law the draw.
template <class Tab>
__device__ __forceinline__ uint64_t delta_cell_t(unsigned long long c, const uint32_t* rk, uint32_t w1, uint32_t w2,
                                                 const Tab& tab, uint64_t ln2_q48, uint64_t inv_lambda, int tie_bits,
                                                 int law) {
    if (law == 4) return delta_of_u(cell_period_q32((uint32_t)c, (uint32_t)(c >> 32), rk, tab, ln2_q48), inv_lambda,
                                    tie_bits);
    return delta_q32_t(w1, w2, tab, ln2_q48, inv_lambda, tie_bits, law);
}

__device__ __forceinline__ uint64_t delta_q32(uint32_t w1, uint32_t w2, const unsigned long long* lr, uint64_t ln2_q48,
                                              uint64_t inv_lambda, int tie_bits, int law = 0) {
    return delta_q32_t(w1, w2, NlogLR{lr}, ln2_q48, inv_lambda, tie_bits, law);
}

// ---------------------------------------------------------------- P7 event hash
// P7 event hash term (docs/PRIMITIVES.md): h = (w3 | 1) * (t ^ (l << 1) ^ s') mod 2^64, w3 the
// fourth Philox word of the arrival's draw, t its time before the increment, l the cell within
// the subarray (0 for the per-cell engines), s' = 1 iff the new spin is +1.
__device__ __forceinline__ uint64_t ev_hash(uint32_t w3, uint64_t t, uint64_t lsb) {
    return (uint64_t)(w3 | 1u) * (t ^ lsb);
}

}  // namespace aca
