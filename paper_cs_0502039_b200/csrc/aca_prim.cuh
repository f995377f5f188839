// aca_prim.cuh — device primitives of the method, implemented from docs/PRIMITIVES.md.
// Shares no code with oracle/ (which implements the same text in plain C).
#pragma once
#include <stdint.h>

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

// ---------------------------------------------------------------- P3 NLOG-2
// -ln(u) in Q32 for u = (X|1)/2^64, integer-only. `lr` points at the interleaved
// {L[i], R[i]} table (shared memory copy of ACA_NLOG_LR).
__device__ __forceinline__ uint64_t nlog_q32(uint64_t X, const unsigned long long* __restrict__ lr,
                                             uint64_t ln2_q48) {
    const uint64_t x = X | 1ull;
    const int z = __clzll((long long)x);
    const uint64_t m = (x << z) << 1;
    const uint32_t i = (uint32_t)(m >> 56);
    const uint64_t g = (m >> 24) & 0xffffffffull;
    const uint64_t Li = lr[2 * i], Ri = lr[2 * i + 1];
    const uint64_t V = (g * Ri) >> 32;                   // < 2^32
    const uint64_t V2 = V * V;
    const uint64_t A = V << 8;
    const uint64_t B = (V2 >> 33) + ((V2 & ((1ull << 33) - 1)) != 0ull);
    const uint32_t C = (uint32_t)(((V2 >> 32) * V) >> 40) / 3u;   // floor(floor(./2^40)/3)
    const uint64_t Wq = (V2 >> 32) + ((V2 & 0xffffffffull) != 0ull);
    const uint64_t W2 = Wq * Wq;
    const uint64_t D = (W2 >> 50) + ((W2 & ((1ull << 50) - 1)) != 0ull);
    const uint64_t lnf = Li + A - B + C - D;
    const uint64_t S = (uint64_t)(z + 1) * ln2_q48 - lnf;
    return (S + (1ull << 15)) >> 16;
}

// Eq. newt1i, next_t > t; P3b tie quantisation.
__device__ __forceinline__ uint64_t delta_q32(uint32_t w1, uint32_t w2, const unsigned long long* lr,
                                              uint64_t ln2_q48, uint64_t inv_lambda, int tie_bits) {
    const uint64_t q = nlog_q32(((uint64_t)w1 << 32) | w2, lr, ln2_q48);
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

// ---------------------------------------------------------------- P7 event hash
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z ^= z >> 30; z *= 0xbf58476d1ce4e5b9ull;
    z ^= z >> 27; z *= 0x94d049bb133111ebull;
    z ^= z >> 31;
    return z;
}
__device__ __forceinline__ uint64_t rotl64(uint64_t v, int r) { return (v << r) | (v >> (64 - r)); }

}  // namespace aca
