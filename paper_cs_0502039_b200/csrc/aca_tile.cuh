// aca_tile.cuh — the production tile path (included by aca_kernels.cuh inside namespace aca).
//
// A persistent CTA per SM runs NG thread groups of NTG threads; each group processes one
// lattice tile at a time, staged with its one-cell halo in shared memory (fig:amcgen's W(c) set,
// the halo is frozen for the visit), runs up to R in-tile rounds of
// fig:s1c1pe per warp and writes the tile back. The CTA owns NBUF > NG tile
// buffers and a fixed, ordered list of tiles; tile k lives in buffer k mod NBUF and is loaded by
// TMA bulk copies (own rows together with their x-halo columns, face rows from the wrapped rows
// or the shard's halo buffers) when the group that processed tile k - NBUF releases the buffer.
// A group that finishes a tile therefore finds its next one already in shared memory: the load
// latency overlaps the other groups' rounds instead of stalling the group.

// Per-lane counters of one tile visit (32-bit: at most NCELL x R x bulk per visit); folded into
// 64-bit totals after every visit (TileTotals).
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

// Per-warp fire queue: CPW/2 + 16 entries (the eligible cells of a warp form an independent
// set: at most one per two cells of each row segment), CPW with a10 candidates.
__host__ __device__ constexpr int tile_queue_per_warp(int cpw, bool early) { return early ? cpw : cpw / 2 + 16; }
// Words of one tile buffer: rows of TX + 4 slots (x-halo at -2..-1 and TX..TX+1, 16-B aligned
// rows for the bulk copies), TY + 2 rows (+ TZ + 2 planes), rounded to 16 words (128 B).
__host__ __device__ constexpr int grp_slots(int ndim, int tx, int ty, int tz) {
    return ((tx + 4) * (ty + 2) * (ndim == 3 ? tz + 2 : 1) + 15) & ~15;
}
// Words (u32) of one spin-bitmap set of the bit-sliced class recount (2-D 64-wide tiles): the even
// and the odd columns' spin bits of the TY rows and the two face rows, and one byte per row
// holding the spins of its two x-halo cells.
__host__ __device__ constexpr int cls_bm_words(int ndim, int tx, int ty) {
    return (ndim == 2 && tx == 64) ? 2 * (ty + 2) + (ty + 3) / 4 + 17 : 0;   // + the deferred count: 16 bins, tile
}
// Shared-memory layout of tile_grp_kernel (host and device): NBUF tile buffers, the P4 (16) and
// a10 (112) tables, the NLOG-2 tables split as L u64[256] and R u32[256], the reduction
// scratch, NBUF mbarriers, 32 u32 of ring control (claim counter, the tile of each group, the
// phases armed on each buffer), the CTA's bounded-lag minimum and T limit (2 u64), the origin
// of the tile in each buffer (32 B each), then the per-warp fire queues.
__host__ __device__ constexpr size_t grp_smem_bytes(int ndim, int tx, int ty, int tz, int ntg, int ng, int nbuf,
                                                    bool early, bool cls = false) {
    return ((size_t)nbuf * grp_slots(ndim, tx, ty, tz) + 16 + 112 + 256 + 128 + (size_t)(ntg * ng) / 32 + nbuf) * 8 +
           160 + 16 + (size_t)nbuf * 64 + (((size_t)(ntg * ng / 32) * tile_queue_per_warp(tx * ty * tz / (ntg / 32), early) * 2 + 15) & ~(size_t)15) +
           (cls ? (size_t)ng * 2 * (16 + cls_bm_words(ndim, tx, ty)) * 4 : 0);
}

// compile-time flag for generic lambdas (one copy of a loop per value)
template <bool B> struct BoolC { static constexpr bool value = B; };

// a10 per-tile class bookkeeping: the BKL class (s, Sigma) of the cell pair (sl, sl + 1) of a
// tile buffer (words v), from the spins of its neighbours in the buffer, added to the per-lane
// class counters (8-bit fields: bins 0-7 in c0, 8-13 in c1; bin = (Sigma + z)/2 + (z + 1)(s + 1)/2
// as the P4 index).
__device__ __forceinline__ void cls_add(uint32_t b, unsigned long long& c0, unsigned long long& c1) {
    const unsigned long long one = 1ull << (8u * (b & 7u));
    if (b < 8u) c0 += one; else c1 += one;
}
template <int NDIM, int SX, int SXY>
__device__ __forceinline__ void cls_pair(const volatile unsigned long long* VS, int sl, ulonglong2 v,
                                         unsigned long long& c0, unsigned long long& c1) {
    constexpr uint32_t Z = 2 * NDIM;
    const uint32_t a = (uint32_t)(v.x & 1ull), b = (uint32_t)(v.y & 1ull);
    const ulonglong2 up = lds128v(&VS[sl - SX]), dn = lds128v(&VS[sl + SX]);
    uint32_t o0 = (uint32_t)(VS[sl - 1] & 1ull) + b + (uint32_t)(up.x & 1ull) + (uint32_t)(dn.x & 1ull);
    uint32_t o1 = a + (uint32_t)(VS[sl + 2] & 1ull) + (uint32_t)(up.y & 1ull) + (uint32_t)(dn.y & 1ull);
    if constexpr (NDIM == 3) {
        const ulonglong2 zl = lds128v(&VS[sl - SXY]), zh = lds128v(&VS[sl + SXY]);
        o0 += (uint32_t)(zl.x & 1ull) + (uint32_t)(zh.x & 1ull);
        o1 += (uint32_t)(zl.y & 1ull) + (uint32_t)(zh.y & 1ull);
    }
    cls_add(o0 + (Z + 1) * a, c0, c1);
    cls_add(o1 + (Z + 1) * b, c0, c1);
}
template <int NDIM, int SX, int SXY>
__device__ __forceinline__ void cls_one(const volatile unsigned long long* VS, int s, unsigned long long w,
                                        unsigned long long& c0, unsigned long long& c1) {
    constexpr uint32_t Z = 2 * NDIM;
    uint32_t o = (uint32_t)(VS[s - 1] & 1ull) + (uint32_t)(VS[s + 1] & 1ull) + (uint32_t)(VS[s - SX] & 1ull) +
                 (uint32_t)(VS[s + SX] & 1ull);
    if constexpr (NDIM == 3) o += (uint32_t)(VS[s - SXY] & 1ull) + (uint32_t)(VS[s + SXY] & 1ull);
    cls_add(o + (Z + 1) * (uint32_t)(w & 1ull), c0, c1);
}
// warp sum of the per-lane counters, added to the group's histogram in shared memory
template <int NBIN>
__device__ __forceinline__ void cls_flush_warp(unsigned long long c0, unsigned long long c1, unsigned int* gh, int lane) {
#pragma unroll
    for (int b = 0; b < NBIN; ++b) {
        const unsigned int v = (unsigned int)(((b < 8 ? c0 : c1) >> (8 * (b & 7))) & 255ull);
        const unsigned int t = __reduce_add_sync(0xffffffffu, v);
        if (lane == 0 && t) atomicAdd(&gh[b], t);
    }
}

// Bit-sliced class count of 32 cells: self = their spin bits, a..d = the spin bits of their
// four neighbours (bit l of every mask belongs to cell l). The neighbour sum k in 0..4 is added
// on bit planes (k = b0 + 2 t0 + 4 t1), then bin k + 5 s gets popc(cells with that k and s):
// the P4 index of (s, Sigma) as in cls_add, for 32 cells in ~35 instructions.
__device__ __forceinline__ void cls_count32(uint32_t self, uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                                            uint32_t* cnt) {
    const uint32_t s1 = a ^ b, c1 = a & b, s2 = c ^ d, c2 = c & d;
    const uint32_t b0 = s1 ^ s2, cy = s1 & s2;
    const uint32_t t0 = c1 ^ c2 ^ cy, t1 = (c1 & c2) | (cy & (c1 ^ c2));
    const uint32_t eq[5] = {~b0 & ~t0 & ~t1, b0 & ~t0 & ~t1, ~b0 & t0 & ~t1, b0 & t0 & ~t1, t1};
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        cnt[k] += __popc(eq[k] & ~self);
        cnt[k + 5] += __popc(eq[k] & self);
    }
}

// A warp's share of the bit-sliced recount of a visit's bitmap set (2-D 64-wide tiles, TY rows
// + 2 face rows): lane l < RPW counts row r0 + l, the warp's bin sums are added to the set's
// deferred histogram (16 u32 after the bitmaps) by lane 0.
template <int TY, int RPW>
__device__ __forceinline__ void cls_count_rows(unsigned int* bm, int r0, int lane) {
    const unsigned char* hb = reinterpret_cast<const unsigned char*>(bm + 2 * (TY + 2));
    unsigned int* dh = bm + 2 * (TY + 2) + (TY + 3) / 4;
    uint32_t cnt[10] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    if (lane < RPW) {
        const int r = r0 + lane;
        const uint32_t E = bm[r + 1], O = bm[TY + 3 + r];
        const uint32_t h = hb[r];
        // even column 2l: left = odd 2l - 1 (the x-halo for l = 0), right = odd 2l
        cls_count32(E, (O << 1) | (h & 1u), O, bm[r], bm[r + 2], cnt);
        // odd column 2l + 1: left = even 2l, right = even 2l + 2 (the x-halo for l = 31)
        cls_count32(O, E, (E >> 1) | ((h >> 1) << 31), bm[TY + 2 + r], bm[TY + 4 + r], cnt);
    }
#pragma unroll
    for (int b = 0; b < 10; ++b) {
        const uint32_t t = __reduce_add_sync(0xffffffffu, cnt[b]);
        if (lane == 0 && t) atomicAdd(&dh[b], t);
    }
}

// Commit the pending arrivals of the cell in slot s for as long as that is exact (a10):
//  * u = 0 (the cell precedes every neighbour): an ordinary arrival, flip iff w0 < thr;
//  * u > 0 neighbours may still change before the arrival: commit it only when the draw
//    rejects the flip for EVERY value of those u spins (w0 >= thm = max threshold over the
//    possible neighbour sums) — "rejected in every consistent world". The arrival then
//    advances t and n and leaves s unchanged, which is what it does in the true trajectory
//    whatever the u neighbours do; the other neighbours' spins are known (they cannot move
//    before the arrival, fig:amcgen stale-read argument PAPER.md:833-871). This is the exact
//    use of the BKL observation that most attempts are rejections.
// thm[(s*(Z+1) + u)*(Z+1) + k] (k = known +1 neighbours) > 2^32 means "wait". u and k come from
// the high halves; a high half equal to the cell's sends the cell to the exact comparison.
template <int NDIM, int SX, int SXY, bool FASTP = false>
__device__ __forceinline__ void commit_loop(const KParams& P, volatile unsigned long long* VS, int s,
                                            unsigned long long cid, uint32_t thr_a, const unsigned long long* thr,
                                            const unsigned long long* thm, const NlogSmem& tab,
                                            unsigned long long wlim, TileStats& st, int gx, int gy, int gz) {
    constexpr int Z = 2 * NDIM;
    const Geo& g = P.g;
    unsigned long long w = VS[s];
    for (int it = 0; it < P.bulk; ++it) {
        if (w >= wlim) break;
        const int off[6] = {-1, 1, -SX, SX, -SXY, SXY};
        uint32_t u = 0, k = 0;
        bool tie = false;
        const unsigned int wh = hi32(w);
#pragma unroll
        for (int q = 0; q < Z; ++q) {
            const unsigned long long nb = VS[s + off[q]];
            const unsigned int nh = hi32(nb);
            const bool below = nh < wh;
            tie = tie || nh == wh;
            u += below;
            k += below ? 0u : (uint32_t)(nb & 1ull);
        }
        if (tie) early_uk<NDIM, SX, SXY>(VS, s, w, g, gx, gy, gz, u, k);
        const uint32_t sb = (uint32_t)(w & 1ull);
        const unsigned long long tm = thm[(sb * (Z + 1) + u) * (Z + 1) + k];
        if (tm > (1ull << 32)) break;                     // must wait for the u neighbours
        const uint32_t n = w_count(w, g);
        if (n == g.nbmask) { atomicOr(&P.ctl->overflow, 1u); break; }
        // FASTP (P.fast: Poisson, lambda = 1, no tie stress, no frames, N < 2^32): the same
        // integers with the general branches compiled out
        const u32x4 r = philox4x32_10_rk(n, (uint32_t)cid, FASTP ? 0u : (uint32_t)(cid >> 32), 0u, P.rk);
        uint32_t flip = 0;
        if (u == 0) flip = (unsigned long long)r.x < thr[k + (uint32_t)(Z + 1) * sb] ? 1u : 0u;
        else if ((unsigned long long)r.x < tm) break;     // a flip is possible in some world: wait
        unsigned long long d;
        if constexpr (FASTP) {
            d = nlog_q32_t(((uint64_t)r.y << 32) | r.z, tab, ACA_LN2_Q48);
            d = d < 1ull ? 1ull : d;
        } else {
            d = delta_cell_t(cid, P.rk, r.y, r.z, tab, ACA_LN2_Q48, P.inv_lambda, P.tie_bits, P.law);
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
    (void)thr_a;
}

// The rounds of one tile visit, per warp (no CTA or group barrier inside: a warp's cells are
// tested and fired by that warp alone; it reads its neighbour warps' boundary rows live, which
// is exact for the same reason as the in-place updates). Each round (fig:s1c1pe): (i) test the
// warp's cells on the 32-bit high halves, (ii) compact the eligible ones with a warp scan,
// (iii) fire them with all lanes busy. A queued cell precedes all its neighbours and none of
// them can pass it before it fires, so its neighbourhood is frozen until it fires.
// Strict rounds decide on strict high-half inequalities only; the last round of a visit, and
// the round after one that found nothing, are exact rounds that also settle high-half ties on
// the full words (lex_lt), so a tied cell waits at most until the end of the visit.
// Lane maps: PAIRMAP (2-D, 64-wide tiles): lane l owns the column pair (2l, 2l+1) of the warp's
// RPW rows and walks them top to bottom with one 128-bit load per row pair, reusing each row as
// the neighbour row of the next (1.5 loads per cell instead of 5). COLMAP (3-D, 32-wide tiles,
// one z-plane per warp): lane l owns column l of the warp's plane. Otherwise lane l owns
// tile-linear cells wbase + l + 32 j.
// GEN: the general arrival (any law, lambda, tie stress, frames, N >= 2^32) is compiled in; without
// it only the fast arrival is (P.fast holds; the host picks the instance per launch), which keeps
// the general path's code out of the production kernel's register allocation.
template <int NDIM, int TX, int TY, int TZ, int NTG, bool FULL, bool EARLY, bool MOORE, bool GEN>
__device__ __forceinline__ unsigned int tile_rounds(const KParams& P, unsigned long long* S, unsigned short* q, int wg,
                                                    uint32_t thr_a, const unsigned long long* thr,
                                                    const unsigned long long* thm, const NlogSmem& tab, int x0, int y0,
                                                    int z0, unsigned long long wlim, TileStats& st) {
    constexpr int SX = TX + 4, SY = TY + 2;
    constexpr int SXY = SX * SY;
    constexpr int NCELL = TX * TY * TZ;
    constexpr int NWG = NTG / 32;
    constexpr int CPW = NCELL / NWG;
    constexpr int JPL = CPW / 32;
    constexpr int Z = MOORE ? 8 : 2 * NDIM;
    constexpr int RPW = CPW / TX > 0 ? CPW / TX : 1;
    constexpr bool FASTMAP = (TX % 32 == 0) && (CPW % TX == 0) && (TY % (CPW / TX > 0 ? CPW / TX : 1) == 0);
    constexpr int LPR = TX / 32 > 0 ? TX / 32 : 1;
    constexpr bool PAIRMAP = FULL && NDIM == 2 && TX == 64 && !MOORE && CPW % TX == 0 && JPL == 2 * RPW && RPW <= 8;
    constexpr bool COLMAP = FULL && NDIM == 3 && TX == 32 && !MOORE && !EARLY && CPW == TX * TY && JPL == TY;
    static_assert(JPL <= 32 && JPL % 4 == 0, "cells per lane");
    const Geo& g = P.g;
    const int lane = threadIdx.x & 31;
    const int wbase = wg * CPW;
    volatile unsigned long long* VS = S;
    const volatile unsigned int* VH = (const volatile unsigned int*)S;   // [2s+1]: high half
    auto slot = [](int lx, int ly, int lz) { return (lz + (NDIM == 3 ? 1 : 0)) * SXY + (ly + 1) * SX + lx + 2; };
    int s0 = 0;
    if (PAIRMAP) {
        s0 = slot(2 * lane, wg * RPW, 0);
    } else if (FASTMAP) {
        const int row0 = wg * RPW;
        s0 = slot(lane, row0 % TY, row0 / TY);
    }
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
    // global coordinates of a tile-local cell (the exact (t, c) comparison needs them)
    auto gcoord = [&](int o, int& gx, int& gy, int& gz) {
        const int lx = o % TX, ly = (o / TX) % TY, lz = o / (TX * TY);
        gx = x0 + lx;
        gy = y0 + ly + (NDIM == 2 ? g.y0 : 0);
        gz = z0 + lz + (NDIM == 3 ? g.z0 : 0);
    };
    auto exact_j = [&](int j, unsigned long long w) {
        int gx, gy, gz;
        gcoord(cell_o(j), gx, gy, gz);
        return exact_min<NDIM, MOORE, SX, SXY>(VS, cell_slot(j), w, g, gx, gy, gz);
    };
    const unsigned int wh = hi32(wlim);
    const bool wexact = (unsigned int)wlim == 0u;   // w < wlim <=> high(w) < high(wlim)
    const bool fastE = EARLY && PAIRMAP && (!GEN || P.fast);   // the a10 fast fire (see the fire step)
    uint32_t fl32 = 0, fi32 = 0;   // fast-path flips / fires (folded into st at the end)
    unsigned int rounds = 0;
    bool exact_next = false;
    for (int r = 0; r < P.rounds; ++r) {
        ACA_TRACE(3, r);
        const bool exact = exact_next || r == P.rounds - 1;
        uint32_t emask = 0;
        int ntest = 0;
        // a10 fast fire (PAIRMAP): the test's decision-table index ti < 50 of each cell j, one byte
        // each (byte j & 3 of pk[j >> 2]; one IMAD per cell for a constant j), carried into its
        // queue entry; the fire step reads u = 0 off ti
        static_assert(!PAIRMAP || JPL <= 16, "a10 index packing: 16 cells per lane");
        uint32_t pk0 = 0u, pk1 = 0u, pk2 = 0u, pk3 = 0u;
        auto pk_set = [&](int j, uint32_t v) {
            const uint32_t add = v << (8 * (j & 3));
            if ((j >> 2) == 0) pk0 += add;
            else if ((j >> 2) == 1) pk1 += add;
            else if ((j >> 2) == 2) pk2 += add;
            else pk3 += add;
        };
        if constexpr (!EARLY && PAIRMAP) {
            unsigned int tiec = ~0u;
            // rows of the lane's column pair, top to bottom; `a` holds row rr, `b` row rr + 1
            // (32-bit shared-window addresses: no generic-to-shared conversion per load)
            const uint32_t sa0 = smem_u32(S) + 8u * (uint32_t)s0;
            const ulonglong2 up = lds128a(sa0 - 8u * SX);
            unsigned int uh0 = hi32(up.x), uh1 = hi32(up.y);
            ulonglong2 a = lds128a(sa0);
// the left / right neighbours' high halves: two 32-bit shared loads at a 16-byte stride (4-way
// bank conflicts: 4 wavefronts each), or (ACA_SHFL_LR, ablation) the neighbour lanes' registers
// by shuffle, the tile's halo columns loaded by lanes 0 and 31 only
#ifdef ACA_SHFL_LR
#define ACA_LR_HALVES                                                                                \
        unsigned int lh = __shfl_up_sync(0xffffffffu, ah1, 1), rh = __shfl_down_sync(0xffffffffu, ah0, 1); \
        if (lane == 0) lh = lds32a(ar - 4u);                                                         \
        if (lane == 31) rh = lds32a(ar + 20u);
#else
#define ACA_LR_HALVES const unsigned int lh = lds32a(ar - 4u), rh = lds32a(ar + 20u);
#endif
#define ACA_PAIR_ROWS(TEST)                                                                          \
    _Pragma("unroll") for (int rr = 0; rr < RPW; ++rr) {                                             \
        const uint32_t ar = sa0 + 8u * SX * (uint32_t)rr;                                            \
        const ulonglong2 b = lds128a(ar + 8u * SX); /* row rr + 1 (the halo row for the last) */     \
        const unsigned int ah0 = hi32(a.x), ah1 = hi32(a.y);                                         \
        ACA_LR_HALVES                                                                                \
        const unsigned int m0 = min(min(lh, ah1), min(uh0, hi32(b.x)));                              \
        const unsigned int m1 = min(min(ah0, rh), min(uh1, hi32(b.y)));                              \
        TEST;                                                                                        \
        uh0 = ah0; uh1 = ah1;                                                                        \
        a = b;                                                                                       \
    }
            if (!exact) {
                ACA_PAIR_ROWS(pair_test_strict(ah0, ah1, m0, m1, wh, 1u << (2 * rr), emask, ntest))
            } else if (wexact) {
                ACA_PAIR_ROWS(pair_test_m(ah0, ah1, m0, m1, wh, 1u << (2 * rr), emask, ntest, tiec))
            } else {
                ACA_PAIR_ROWS(pair_test(ah0, ah1, m0, m1, wh, 1u << (2 * rr), emask, ntest, tiec))
            }
#undef ACA_PAIR_ROWS
            if (tiec == 0u) {   // rare: exact test of the lane's cells
                emask = 0;
                ntest = 0;
#pragma unroll 1
                for (int j = 0; j < JPL; ++j) {
                    const unsigned long long w = VS[cell_slot(j)];
                    if (w >= wlim) continue;
                    ++ntest;
                    if (exact_j(j, w)) emask |= 1u << j;
                }
            }
        } else if constexpr (!EARLY && COLMAP) {
            unsigned int tiec = ~0u;
            // high halves only, through 32-bit shared-window addresses (byte offset +4 of a word)
            const uint32_t ha0 = smem_u32(S) + 8u * (uint32_t)s0 + 4u;
            unsigned int uh = lds32a(ha0 - 8u * SX);
            unsigned int ah_ = lds32a(ha0);
#define ACA_COL_ROWS(TEST)                                                                           \
    _Pragma("unroll") for (int rr = 0; rr < TY; ++rr) {                                              \
        const uint32_t hr = ha0 + 8u * SX * (uint32_t)rr;                                            \
        const unsigned int bh = lds32a(hr + 8u * SX);                                                \
        const unsigned int ah = ah_;                                                                 \
        const unsigned int m = min(min(min(lds32a(hr - 8u), lds32a(hr + 8u)),                        \
                                       min(lds32a(hr - 8u * SXY), lds32a(hr + 8u * SXY))),           \
                                   min(uh, bh));                                                     \
        TEST;                                                                                        \
        uh = ah;                                                                                     \
        ah_ = bh;                                                                                    \
    }
            if (!exact) {
                ACA_COL_ROWS(one_test_strict(ah, m, wh, 1u << rr, emask, ntest))
            } else if (wexact) {
                ACA_COL_ROWS(one_test_m(ah, m, wh, 1u << rr, emask, ntest, tiec))
            } else {
                ACA_COL_ROWS(one_test(ah, m, wh, 1u << rr, emask, ntest, tiec))
            }
#undef ACA_COL_ROWS
            if (tiec == 0u) {
                emask = 0;
                ntest = 0;
#pragma unroll 1
                for (int j = 0; j < JPL; ++j) {
                    const unsigned long long w = VS[cell_slot(j)];
                    if (w >= wlim) continue;
                    ++ntest;
                    if (exact_j(j, w)) emask |= 1u << j;
                }
            }
        } else if constexpr (!EARLY) {
            // generic map: exact every round; batches of 4 cells, every load of a batch issued
            // before any compare, tied high halves settled on the full words
            uint32_t tmask = 0, amask = 0;
#pragma unroll
            for (int j0 = 0; j0 < JPL; j0 += 4) {
                unsigned long long wv[4];
                unsigned int mv[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) wv[k] = VS[cell_slot(j0 + k)];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
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
                for (int k = 0; k < 4; ++k) {
                    const bool act = cell_valid(j0 + k) && wv[k] < wlim;
                    const unsigned int oh = hi32(wv[k]);
                    emask |= (uint32_t)(act && oh < mv[k]) << (j0 + k);
                    tmask |= (uint32_t)(act && oh == mv[k]) << (j0 + k);
                    amask |= (uint32_t)act << (j0 + k);
                }
            }
            while (tmask) {   // tie in the high halves: decide on the full words
                const int j = __ffs(tmask) - 1;
                tmask &= tmask - 1u;
                emask |= (uint32_t)exact_j(j, VS[cell_slot(j)]) << j;
            }
            ntest = __popc(amask);
        } else if constexpr (PAIRMAP) {
            // a10 with the column-pair walk: the four neighbours' words are in registers, so u
            // (neighbours before the cell) and k (+1 spins among the others) come from one pass
            // on the high halves; u = 0 is the local minimum, else the a10 table decides. A
            // neighbour whose high half equals the cell's sends the lane to the exact pass.
            unsigned int tiec = ~0u;
            const ulonglong2 up = lds128v(&VS[s0 - SX]);
            unsigned long long u0 = up.x, u1 = up.y;
            ulonglong2 a = lds128v(&VS[s0]);
            // table index ti = 25 s + 5 u + k = 25 s + sum over neighbours of (before ? 5 : spin
            // bit); the candidate test is one bit of the mask built at kernel start (thm[100])
            static_assert(Z == 4, "a10 PAIRMAP index");
            const unsigned long long cmask = thm[100];
            // Strict rounds count a neighbour with an equal high half as one that may come before
            // (unknown): conservative for the rejection test, and u = 0 still means a strict local
            // minimum; exact rounds send such lanes to the exact pass instead.
            auto early_cell = [&](bool strict, unsigned long long w, unsigned long long n0, unsigned long long n1,
                                  unsigned long long n2, unsigned long long n3, int j) {
                if (w >= wlim) return;
                ++ntest;
                const unsigned int h = hi32(w), h0 = hi32(n0), h1 = hi32(n1), h2 = hi32(n2), h3 = hi32(n3);
                uint32_t v;
                if (strict) {
                    v = (h0 <= h ? 5u : (uint32_t)n0 & 1u) + (h1 <= h ? 5u : (uint32_t)n1 & 1u) +
                        (h2 <= h ? 5u : (uint32_t)n2 & 1u) + (h3 <= h ? 5u : (uint32_t)n3 & 1u);
                } else {
                    if (h0 == h || h1 == h || h2 == h || h3 == h) tiec = 0u;
                    v = (h0 < h ? 5u : (uint32_t)n0 & 1u) + (h1 < h ? 5u : (uint32_t)n1 & 1u) +
                        (h2 < h ? 5u : (uint32_t)n2 & 1u) + (h3 < h ? 5u : (uint32_t)n3 & 1u);
                }
                const uint32_t ti = (uint32_t)(w & 1ull) * 25u + v;
                emask |= (uint32_t)((cmask >> ti) & 1ull) << j;
                if (fastE) pk_set(j, ti);
            };
#define ACA_EARLY_ROWS(STRICT)                                                                       \
    _Pragma("unroll") for (int rr = 0; rr < RPW; ++rr) {                                             \
        const int sr = s0 + rr * SX;                                                                 \
        const ulonglong2 b = lds128v(&VS[sr + SX]);                                                  \
        const unsigned long long lw = VS[sr - 1], rw = VS[sr + 2];                                   \
        early_cell(STRICT, a.x, lw, a.y, u0, b.x, 2 * rr);                                           \
        early_cell(STRICT, a.y, a.x, rw, u1, b.y, 2 * rr + 1);                                       \
        u0 = a.x; u1 = a.y;                                                                          \
        a = b;                                                                                       \
    }
            if (!exact) {
                ACA_EARLY_ROWS(true)
            } else {
                ACA_EARLY_ROWS(false)
            }
#undef ACA_EARLY_ROWS
            if (tiec == 0u) {
                emask = 0;
                ntest = 0;
                pk0 = pk1 = pk2 = pk3 = 0u;   // the first pass's indices are replaced, not merged
#pragma unroll 1
                for (int j = 0; j < JPL; ++j) {
                    const int sj = cell_slot(j);
                    const unsigned long long w = VS[sj];
                    if (w >= wlim) continue;
                    ++ntest;
                    int gx, gy, gz;
                    gcoord(cell_o(j), gx, gy, gz);
                    uint32_t u, k;
                    early_uk<NDIM, SX, SXY>(VS, sj, w, g, gx, gy, gz, u, k);
                    const uint32_t ti = ((uint32_t)(w & 1ull) * (Z + 1) + u) * (Z + 1) + k;
                    const bool e = u == 0u || thm[ti] <= (1ull << 32);
                    emask |= (uint32_t)e << j;
                    if (fastE) pk_set(j, ti);
                }
            }
        } else {
            // generic a10 test: exact (t, c) comparisons per cell (ragged tiles, other maps)
#pragma unroll 1
            for (int j = 0; j < JPL; ++j) {
                if (!cell_valid(j)) continue;
                const int sj = cell_slot(j);
                const unsigned long long w = VS[sj];
                if (w >= wlim) continue;
                ++ntest;
                int gx, gy, gz;
                gcoord(cell_o(j), gx, gy, gz);
                uint32_t u, k;
                early_uk<NDIM, SX, SXY>(VS, sj, w, g, gx, gy, gz, u, k);
                const bool e = u == 0u || thm[((uint32_t)(w & 1ull) * (Z + 1) + u) * (Z + 1) + k] <= (1ull << 32);
                emask |= (uint32_t)e << j;
            }
        }
        st.tested += ntest;
        // compaction: warp-exclusive scan of the per-lane counts, then each lane writes its
        // eligible cells' tile-local indices into the warp's queue
        const int mine = __popc(emask);
        int incl = mine;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += v;
        }
        const int cnt = __shfl_sync(0xffffffffu, incl, 31);
        const int pos = incl - mine;
        ACA_CHECK(cnt <= tile_queue_per_warp(CPW, EARLY), cnt, wg);
        ACA_TRACE(4, ((unsigned long long)cnt << 8) | r);
        if constexpr (PAIRMAP) {
            // entry of cell j = base + (j / 2) TX + j % 2 = base | ((j << 5) & 0x1c0) | (j & 1)
            // (base = warp CPW + 2 lane has no bits in 0x1c1); highest bit first
            static_assert(!PAIRMAP || (TX == 64 && RPW <= 8), "PAIRMAP entry packing");
            uint32_t qp = smem_u32(q) + 2u * (uint32_t)pos;
            const uint32_t base = (uint32_t)(wbase + 2 * lane);
            while (emask) {
                uint32_t j;
                asm("bfind.u32 %0, %1;" : "=r"(j) : "r"(emask));
                emask ^= 1u << j;
                uint32_t e;
                if (EARLY && fastE) {   // warp-local cell (9 bits) | table index (6 bits)
                    const uint32_t ti = __byte_perm(j < 8u ? pk0 : pk2, j < 8u ? pk1 : pk3, j & 7u) & 0xffu;
                    e = (uint32_t)(2 * lane) | ((j << 5) & 0x1c0u) | (j & 1u) | (ti << 9);
                } else {
                    e = base | ((j << 5) & 0x1c0u) | (j & 1u);
                }
                asm volatile("st.shared.u16 [%0], %1;" ::"r"(qp), "h"((unsigned short)e) : "memory");
                qp += 2u;
            }
        } else if constexpr (COLMAP) {
            // entry of cell j = wbase + lane + 32 j
            uint32_t qp = smem_u32(q) + 2u * (uint32_t)pos;
            const uint32_t base = (uint32_t)(wbase + lane);
            while (emask) {
                uint32_t j;
                asm("bfind.u32 %0, %1;" : "=r"(j) : "r"(emask));
                emask ^= 1u << j;
                asm volatile("st.shared.u16 [%0], %1;" ::"r"(qp), "h"((unsigned short)(base + (j << 5))) : "memory");
                qp += 2u;
            }
        } else {
            int p = pos;
            while (emask) {
                const int j = __ffs(emask) - 1;
                emask &= emask - 1u;
                q[p++] = (unsigned short)cell_o(j);
            }
        }
        __syncwarp();
        if (EARLY && PAIRMAP && fastE) {
            // a10 on 64-wide 2-D tiles with the fast arrival: each entry carries its cell's
            // decision-table index from the test. Using the test-time (u, k) is exact: a neighbour
            // that came after the cell then cannot change before the cell's arrival (it is not a
            // local minimum while the cell precedes it), and one that came before stays counted
            // as unknown even if it has fired since (commit_loop's rule, on an older snapshot).
            const uint32_t qa = smem_u32(q), sa = smem_u32(S), ta = smem_u32(thm);
            const uint32_t cb = (uint32_t)(y0 + g.y0) * (uint32_t)g.nx + (uint32_t)x0;
            for (int i = lane; i < cnt; i += 32) {
                uint32_t e;
                asm volatile("ld.shared.u16 %0, [%1];" : "=r"(e) : "r"(qa + 2u * (uint32_t)i) : "memory");
                const uint32_t o = (uint32_t)wbase + (e & 511u);
                const uint32_t lx = o % TX, ly = o / TX;
                const uint32_t a = sa + 8u * (uint32_t)slot((int)lx, (int)ly, 0);
                unsigned long long w, tm;
                asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(w) : "r"(a) : "memory");
                const uint32_t ti = (e >> 9) & 63u;
                asm volatile("ld.shared.u64 %0, [%1];" : "=l"(tm) : "r"(ta + 8u * ti));
                const uint32_t n = w_count(w, g);
                if (n == g.nbmask) { atomicOr(&P.ctl->overflow, 1u); continue; }
                const u32x4 rr = philox4x32_10_rk(n, cb + ly * (uint32_t)g.nx + lx, 0u, 0u, P.rk);
                const bool lo = (unsigned long long)rr.x < tm;
                // u = 0 iff ti mod 25 < 5: bits 0-4 and 25-29 of 0x3e00001f (clamped shift: 0 for ti >= 32)
                const bool u0 = (__funnelshift_rc(0x3e00001fu, 0u, ti) & 1u) != 0u;
                if (lo && !u0) continue;   // u > 0 and a flip is possible in some world: wait
                const uint32_t flip = lo ? 1u : 0u;    // u = 0: the P4 decision; u > 0: rejected in every world
                unsigned long long d = nlog_q32_t(((uint64_t)rr.y << 32) | rr.z, tab, ACA_LN2_Q48);
                d = d < 1ull ? 1ull : d;
                if (P.do_hash) st.hacc += ev_hash(rr.w, w >> g.TSH, (unsigned long long)((uint32_t)(w & 1ull) ^ flip));
                const unsigned long long wn = (w + (d << g.TSH) + 2ull) ^ (unsigned long long)flip;
                asm volatile("st.volatile.shared.u64 [%0], %1;" ::"r"(a), "l"(wn) : "memory");
                fl32 += flip;
                ++fi32;
            }
        } else if ((PAIRMAP || COLMAP) && !EARLY && (!GEN || P.fast)) {
            // The common case (64-wide 2-D / 32-wide 3-D tiles, Poisson, lambda = 1, no frames):
            // the queue, the words and the tables are addressed with 32-bit shared-window offsets.
            const uint32_t qa = smem_u32(q), sa = smem_u32(S);
            const uint32_t cb = NDIM == 2 ? (uint32_t)(y0 + g.y0) * (uint32_t)g.nx + (uint32_t)x0 : 0u;
            for (int i = lane; i < cnt; i += 32) {
                uint32_t o;
                asm volatile("ld.shared.u16 %0, [%1];" : "=r"(o) : "r"(qa + 2u * (uint32_t)i) : "memory");
                ACA_CHECK(o < (uint32_t)NCELL, o, i);
                if (!ACA_DBG_OK(o < (uint32_t)NCELL)) continue;
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
                const FireOut f = fire_fast(w, ones, Z, cid, g, thr_a, tab, P.rk, P.do_hash);
                if (!f.ok) { atomicOr(&P.ctl->overflow, 1u); continue; }
                asm volatile("st.volatile.shared.u64 [%0], %1;" ::"r"(a), "l"(f.wnew) : "memory");
                st.hacc += f.h;
                fl32 += f.flip;
                ++fi32;
            }
        } else {
            for (int i = lane; i < cnt; i += 32) {
                const int o = q[i];
                ACA_CHECK(o >= 0 && o < NCELL, o, i);
                if (!ACA_DBG_OK(o >= 0 && o < NCELL)) continue;
                const int lx = o % TX, ly = (o / TX) % TY, lz = o / (TX * TY);
                const int s = slot(lx, ly, lz);
                ACA_CHECK(s >= SX && s < SXY * (NDIM == 3 ? TZ + 2 : 1) - SX, s, o);
                if (EARLY) {
                    int gx, gy, gz;
                    gcoord(o, gx, gy, gz);
                    if (!GEN || P.fast)
                        commit_loop<NDIM, SX, SXY, true>(P, VS, s, cell_id32t<NDIM>(g, x0 + lx, y0 + ly, z0 + lz), thr_a,
                                                         thr, thm, tab, wlim, st, gx, gy, gz);
                    else if constexpr (GEN)
                        commit_loop<NDIM, SX, SXY>(P, VS, s, cell_id(g, x0 + lx, y0 + ly, z0 + lz), thr_a, thr, thm,
                                                   tab, wlim, st, gx, gy, gz);
                    continue;
                }
                const unsigned long long w = VS[s];
                uint32_t ones = (VH[2 * (s - 1)] & 1u) + (VH[2 * (s + 1)] & 1u) + (VH[2 * (s - SX)] & 1u) +
                                (VH[2 * (s + SX)] & 1u);
                if (NDIM == 3) ones += (VH[2 * (s - SXY)] & 1u) + (VH[2 * (s + SXY)] & 1u);
                if (MOORE)
                    ones += (VH[2 * (s - SX - 1)] & 1u) + (VH[2 * (s - SX + 1)] & 1u) + (VH[2 * (s + SX - 1)] & 1u) +
                            (VH[2 * (s + SX + 1)] & 1u);
                if (!GEN || P.fast) {   // Poisson law, lambda = 1, no tie stress, no frames, N < 2^32
                    const FireOut f = fire_fast(w, ones, Z, cell_id32t<NDIM>(g, x0 + lx, y0 + ly, z0 + lz), g, thr_a,
                                                tab, P.rk, P.do_hash);
                    if (!f.ok) { atomicOr(&P.ctl->overflow, 1u); continue; }
                    VS[s] = f.wnew;
                    st.hacc += f.h;
                    fl32 += f.flip;
                    ++fi32;
                    continue;
                }
                if constexpr (GEN) {
                    const FireOut f = fire(w, ones, Z, cell_id(g, x0 + lx, y0 + ly, z0 + lz), g, thr, tab, P.rk,
                                           P.inv_lambda, P.tie_bits, P.do_hash, P.ctl, P.law, &P.fr);
                    if (!f.ok) continue;
                    VS[s] = f.wnew;
                    st.hacc += f.h;
                    st.flips += f.flip;
                    ++st.fired;
                }
            }
        }
        ACA_TRACE(5, r);
        // Every queued cell's new word must be visible to the whole warp before its next test:
        // a queued cell is still a local minimum until its word is written, and lanes of a warp
        // are not guaranteed to reconverge after the divergent fire loop.
        __syncwarp();
        ++rounds;
        if (cnt == 0) {
            if (exact) break;      // nothing eligible, ties included: this warp is done
            exact_next = true;     // settle possible high-half ties before giving up
        } else {
            exact_next = false;
        }
    }
    st.flips += fl32;
    st.fired += fi32;
    return rounds;
}

// ------------------------------------------------------------ grouped persistent tile kernel
// EM: 0 = the plain test; 1 = the a10 path on every tile; 2 = per-tile class bookkeeping (a10 as
// north_star words it): every visit recounts the BKL classes of the tile's cells at its
// write-back into P.tile_hist, and the next visit of the tile takes the a10 path iff the tile's
// n-fold flip weight sum_k |Gamma_k| p_k is at most P.cls_lim.
template <int NDIM, int TX, int TY, int TZ, int NTG, int NG, int NBUF, int EM, bool MOORE, bool GEN>
__global__ void __launch_bounds__(NTG * NG, 1) tile_grp_kernel(const __grid_constant__ KParams P) {
    constexpr bool EARLY = EM != 0;   // queue sizing: a10 candidates
    constexpr bool CLS = EM == 2;
    constexpr int NBIN = 2 * (2 * NDIM + 1);
    static_assert(!MOORE || NDIM == 2, "Moore neighbourhood: 2-D");
    static_assert(NG >= 1 && NG <= 14 && NBUF >= 1 && 1 + 2 * NG + NBUF <= 30, "groups / buffers");
    constexpr int NT = NTG * NG;
    constexpr int SX = TX + 4, SY = TY + 2, SZ = (NDIM == 3) ? TZ + 2 : 1;
    constexpr int SXY = SX * SY;
    constexpr int NSLOT = SXY * SZ;
    constexpr int NSLOTP = grp_slots(NDIM, TX, TY, TZ);
    constexpr int NCELL = TX * TY * TZ;
    constexpr int NROWS = TY * TZ;
    constexpr int NWG = NTG / 32;
    constexpr int NW = NT / 32;
    constexpr int CPW = NCELL / NWG;
    constexpr int NFACE = NDIM == 2 ? 2 : 2 * TY + 2 * TZ;
    constexpr int QW = tile_queue_per_warp(CPW, EARLY);
    static_assert(NCELL % NTG == 0 && CPW % 32 == 0 && TX % 4 == 0, "tile/group mismatch");

    if (*(volatile unsigned int*)&P.ctl->done) return;

    extern __shared__ __align__(128) unsigned long long smem[];
    unsigned long long* Sb = smem;                          // NBUF x NSLOTP words
    unsigned long long* thr = Sb + NBUF * NSLOTP;           // 16
    unsigned long long* thm = thr + 16;                     // 112 (a10 table)
    unsigned long long* Lt = thm + 112;                     // 256 (NLOG-2 L)
    unsigned int* Rt = (unsigned int*)(Lt + 256);           // 256 u32 (NLOG-2 R, low words)
    unsigned long long* red = Lt + 256 + 128;               // NW
    unsigned long long* bar = red + NW;                     // NBUF full barriers
    unsigned int* cs = (unsigned int*)(bar + NBUF);         // [0] claim counter, [1 + 2g + p] tiles of group g
    volatile unsigned int* armed = cs + 1 + 2 * NG;         // [b] phases of bar[b] armed so far
    unsigned long long* lagw = (unsigned long long*)(cs + 32);   // [0] bounded lag: min word written back, [1] wlim_T
    int4* orgs = (int4*)(((uintptr_t)(cs + 40) + 15) & ~(uintptr_t)15);   // [2s], [2s+1]: origin of tile k, s = k % (2 NBUF)
    unsigned short* Q = (unsigned short*)(orgs + 4 * NBUF); // NW x QW fire queue entries
    // CLS: per group two 16-bin class histograms (the visit in progress, by the parity `par`)
    unsigned int* ghist = (unsigned int*)((char*)Q + (((size_t)NW * QW * 2 + 15) & ~(size_t)15));
    // CLS on 2-D 64-wide tiles: the fast tiles' classes are recounted from spin bitmaps built by
    // ballots at the write-back (per group two sets, by the parity `par`), the others per cell
    constexpr int CBMW = cls_bm_words(NDIM, TX, TY);
    constexpr bool BMC = CLS && CBMW > 0 && (NCELL / NWG) % TX == 0;
    unsigned int* cbm = ghist + NG * 32;

    const Geo& g = P.g;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gid = tid / NTG, gt = tid - gid * NTG, wg = gt >> 5;
    if (tid < 16) thr[tid] = tid < 14 ? P.thr[tid] : 0ull;
    for (int i = tid; i < 112; i += NT) {
        unsigned long long v = i < 98 ? P.thm[i] : ~0ull;
        if (NDIM == 2 && i == 100) {   // 2-D a10 candidate mask: bit ti <=> u = 0 or thm[ti] <= 2^32
            v = 0ull;
            for (int t = 0; t < 50; ++t)
                if (t % 25 < 5 || P.thm[t] <= (1ull << 32)) v |= 1ull << t;
        }
        thm[i] = v;
    }
    for (int i = tid; i < 256; i += NT) {
        Lt[i] = P.lr[2 * i];
        Rt[i] = (unsigned int)P.lr[2 * i + 1];
    }
    if (tid < NBUF) { mbar_init(&bar[tid], 1); armed[tid] = 0u; }
    if constexpr (CLS)
        for (int i = tid; i < NG * 32; i += NT) ghist[i] = 0u;
    if constexpr (BMC)
        for (int i = tid; i < NG * 2 * 17; i += NT) {   // deferred counts: bins 0, tile -1
            unsigned int* dh = cbm + (i / 17) * CBMW + 2 * (TY + 2) + (TY + 3) / 4;
            dh[i % 17] = i % 17 == 16 ? ~0u : 0u;
        }
    if (tid == 0) {
        cs[0] = 0u;
        cs[30] = cs[31] = 0u;   // CLS: tile visits per path
        lagw[0] = ~0ull;
        lagw[1] = *(volatile unsigned long long*)&P.ctl->wlim_T;
    }
    __syncthreads();
    const NlogSmem tab{smem_u32(Lt), smem_u32(Rt)};
    const uint32_t thr_a = smem_u32(thr);

    auto slot = [](int lx, int ly, int lz) { return (lz + (NDIM == 3 ? 1 : 0)) * SXY + (ly + 1) * SX + lx + 2; };
    const unsigned long long wlim = *(volatile unsigned long long*)&P.ctl->wlim;      // firing limit
    // work items: every tile (phase < 0), or the tiles of one checkerboard colour: item k is
    // column pair j = k % hx of tile row k / hx, tx = 2j + ((row parity + phase) & 1)
    const int hx = (P.tiles_x + 1) >> 1;
    const int ntiles = P.phase < 0 ? P.tiles_x * P.tiles_y * P.tiles_z : hx * P.tiles_y * P.tiles_z;
    const int K = (int)blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const bool vec_ok = (g.nx % 2) == 0;
    const bool reverse = P.phase < 0 && ((*(volatile unsigned long long*)&P.ctl->launches) & 1ull);

    struct Org { int x0, y0, z0, tx, ty, tz; bool valid, full, early; };
    auto origin = [&](int k) -> Org {
        const int it = (int)blockIdx.x + k * (int)gridDim.x;
        Org o;
        if (P.phase < 0) {
            const int tile = reverse ? ntiles - 1 - it : it;
            o.tx = tile % P.tiles_x; o.ty = (tile / P.tiles_x) % P.tiles_y; o.tz = tile / (P.tiles_x * P.tiles_y);
        } else {
            const int row = it / hx;
            o.ty = row % P.tiles_y; o.tz = row / P.tiles_y;
            o.tx = 2 * (it % hx) + ((o.ty + o.tz + P.row_par0 + P.phase) & 1);
        }
        o.x0 = o.tx * TX; o.y0 = o.ty * TY; o.z0 = o.tz * TZ;
        o.valid = o.tx < P.tiles_x;   // odd tiles_x: the last column pair has one tile
        o.full = o.valid && o.x0 + TX <= g.nx && o.y0 + TY <= g.ny && (NDIM == 2 || o.z0 + TZ <= g.nz);
        o.early = EM == 1;
        return o;
    };
    auto tile_index = [&](const Org& o) { return ((size_t)o.tz * P.tiles_y + o.ty) * P.tiles_x + o.tx; };
    // Which staged words may another writer store while we copy them? Own rows: nobody (a tile
    // is processed by one group per launch). In a checkerboard launch the tiles adjacent to
    // ours have the other colour and are idle, except across a periodic wrap with an odd tile
    // count; halo buffers of a peer process are written concurrently. Words with a possible
    // concurrent writer are read by threads with single-copy-atomic relaxed 8-byte loads; the
    // rest by TMA bulk copies (whose atomicity is only per copy).
    auto wrap_safe = [&](int t, int nt_axis) { return nt_axis == 1 || (nt_axis & 1) == 0 || (t != 0 && t != nt_axis - 1); };
    auto x_tma = [&](const Org& o) { return P.phase >= 0 && wrap_safe(o.tx, P.tiles_x); };
    // face row f (2-D: 0 = y0 - 1, 1 = y0 + TY; 3-D: z faces 0..2TY-1, then y faces)
    auto face_coords = [&](int f, int& ly, int& lz) {
        if (NDIM == 2) { ly = f == 0 ? -1 : TY; lz = 0; }
        else if (f < 2 * TY) { lz = f < TY ? -1 : TZ; ly = f % TY; }
        else { const int f2 = f - 2 * TY; ly = f2 < TZ ? -1 : TY; lz = f2 % TZ; }
    };
    auto face_ok = [&](const Org& o, bool zface, bool lo) {
        const int t = zface ? o.tz : o.ty, nt_axis = zface ? P.tiles_z : P.tiles_y;
        const bool wraps = lo ? t == 0 : t == nt_axis - 1;
        const bool sharded_axis = NDIM == 2 || zface;
        if (wraps && sharded_axis && g.sharded) return !P.halo_peer;   // a halo buffer
        return P.phase >= 0 && (!wraps || wrap_safe(t, nt_axis));
    };
    auto face_tma = [&](const Org& o, int f) {
        if (NDIM == 2) return face_ok(o, false, f == 0);
        if (f < 2 * TY) return face_ok(o, true, f < TY);
        return face_ok(o, false, f - 2 * TY < TZ);
    };
    auto face_rows_tma = [&](const Org& o) {
        if (NDIM == 2) return (int)face_ok(o, false, true) + (int)face_ok(o, false, false);
        return TY * ((int)face_ok(o, true, true) + (int)face_ok(o, true, false)) +
               TZ * ((int)face_ok(o, false, true) + (int)face_ok(o, false, false));
    };
    // Staging of tile k into buffer b in two steps. arm (one thread): announce the bytes the
    // bulk copies will deliver on bar[b] (or just arrive, for a tile that is not all-TMA, so the
    // phases stay aligned with the tile count) and publish that phase k / NBUF is armed.
    // copy_rows (every thread of a group or warp, `t` of `nt`): issue the row copies.
    // The origin of the tile in buffer b is computed once (integer divisions by runtime tile
    // counts) by the arming thread and read by everyone else from shared memory.
    // The origin of tile k lives in slot k % (2 NBUF), not in its buffer's slot: a warp of the
    // group processing tile k may read it after the group's thread 0 has armed tile k + NBUF (same
    // buffer) — the arm precedes the visit's closing barrier, not its opening.
    auto org_load = [&](int k) -> Org {
        const int os = k % (2 * NBUF);
        const int4 a = orgs[2 * os], c = orgs[2 * os + 1];
        Org o;
        o.x0 = a.x; o.y0 = a.y; o.z0 = a.z; o.tx = a.w; o.ty = c.x; o.tz = c.y; o.valid = c.z != 0;
        o.full = (c.w & 1) != 0;
        o.early = EM == 1 || (c.w & 2) != 0;
        return o;
    };
    auto box_ok = [&](const Org& o) {
        if (!P.box_ok || P.phase < 0 || !(o.full && vec_ok)) return false;
        if (o.x0 < 2 || o.x0 + TX + 2 > g.nx || o.y0 < 1 || o.y0 + TY + 1 > g.ny) return false;
        return NDIM == 2 || (o.z0 >= 1 && o.z0 + TZ + 1 <= g.nz);
    };
    constexpr uint32_t BOX_BYTES = (uint32_t)(TX + 4) * (TY + 2) * (NDIM == 3 ? TZ + 2 : 1) * 8u;
    auto arm = [&](int k, int b) {
        const Org o = origin(k);
        bool early = false;
        if constexpr (CLS) {   // the tile's classes at its last visit decide its path for this one
#ifdef ACA_ABL_NOARM
            if (false) {
#else
            if (o.valid) {
#endif
                const uint4* hp = reinterpret_cast<const uint4*>(P.tile_hist + 16 * tile_index(o));
                long long wsum = 0;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint4 v = hp[j];
                    wsum += (long long)v.x * P.clsw[4 * j] + (long long)v.y * P.clsw[4 * j + 1] +
                            (long long)v.z * P.clsw[4 * j + 2] + (long long)v.w * P.clsw[4 * j + 3];
                }
                early = wsum <= P.cls_lim;
            }
        }
        const int os = k % (2 * NBUF);
        orgs[2 * os] = make_int4(o.x0, o.y0, o.z0, o.tx);
        orgs[2 * os + 1] = make_int4(o.ty, o.tz, o.valid ? 1 : 0, (o.full ? 1 : 0) | (early ? 2 : 0));
        const bool fast = o.full && vec_ok;
        if (box_ok(o)) {
            mbar_arrive_expect_tx(&bar[b], BOX_BYTES);
        } else if (fast) {
            const int rw = x_tma(o) ? TX + 4 : TX;       // words per staged row
            mbar_arrive_expect_tx(&bar[b], (uint32_t)((NROWS + face_rows_tma(o)) * rw * 8));
        } else {
            mbar_arrive(&bar[b]);
        }
        __threadfence_block();
        armed[b] = (unsigned int)(k / NBUF) + 1u;   // phase k / NBUF of bar[b] is armed
    };
    auto copy_rows = [&](int k, int t, int nt) {   // tile k, after arm(k, k % NBUF) is visible to the caller
        const int b = k % NBUF;
        const Org o = org_load(k);
        if (!(o.full && vec_ok)) return;
        const bool xs = x_tma(o);
        unsigned long long* S = Sb + b * NSLOTP;
        const uint32_t barA = smem_u32(&bar[b]);
        if (box_ok(o)) {
            if (t == 0) {
                fence_proxy_async();
                if constexpr (NDIM == 2) tma_box_2d(smem_u32(S), &P.tmap, o.x0 - 2, o.y0 - 1, barA);
                else tma_box_3d(smem_u32(S), &P.tmap, o.x0 - 2, o.y0 - 1, o.z0 - 1, barA);
            }
            return;
        }
        bool fenced = false;
        for (int row = t; row < NROWS + NFACE; row += nt) {
            int ly, lz;
            const unsigned long long* rowp;
            if (row < NROWS) {
                ly = row % TY; lz = row / TY;
                rowp = NDIM == 2 ? P.words + (size_t)(o.y0 + ly) * g.nx
                                 : P.words + ((size_t)(o.z0 + lz) * g.ny + (o.y0 + ly)) * g.nx;
            } else {
                if (!face_tma(o, row - NROWS)) continue;
                face_coords(row - NROWS, ly, lz);
                rowp = word_ptr_t<true>(P, 0, o.y0 + ly, o.z0 + lz);
            }
            if (!fenced) { fence_proxy_async(); fenced = true; }
            unsigned long long* d0 = &S[slot(0, ly, lz)];
            ACA_CHECK(slot(-2, ly, lz) >= 0 && slot(TX + 2, ly, lz) <= NSLOTP, row, ly);
            ACA_CHECK(rowp != nullptr && ((uintptr_t)rowp & 15) == 0, (uintptr_t)rowp, row);
            const uint32_t da = smem_u32(d0);
            if (!xs) {
                bulk_g2s_a(da, rowp + o.x0, TX * 8, barA);
                continue;
            }
            // columns x0-2 .. x0+TX+1; the parts across the periodic x wrap come separately
            const bool lo_in = o.x0 >= 2, hi_in = o.x0 + TX + 2 <= g.nx;
            const int st = lo_in ? o.x0 - 2 : o.x0, en = hi_in ? o.x0 + TX + 2 : o.x0 + TX;
            bulk_g2s_a(da + 8u * (uint32_t)(st - o.x0), rowp + st, (uint32_t)(en - st) * 8u, barA);
            if (!lo_in) bulk_g2s_a(da - 16u, rowp + g.nx - 2, 16u, barA);
            if (!hi_in) bulk_g2s_a(da + 8u * TX, rowp, 16u, barA);
        }
    };

    if (warp == 0) {   // the first NBUF tiles of this CTA
        for (int k = 0; k < NBUF && k < K; ++k) {
            if (lane == 0) arm(k, k);
            __syncwarp();
            copy_rows(k, lane, 32);
        }
    }


    TileStats st;
    TileTotals tot;
    unsigned int active = 0;   // cells of this CTA still below T (< 2^32: N < 2^32)
    unsigned int rounds_max = 0;
    unsigned short* q = Q + warp * QW;
    // A group's next tile is claimed by its thread 0 before the write-back barrier that ends
    // the current one, into the other of the group's two slots (everybody has read the current
    // slot by then), so one group barrier per tile visit suffices when no thread patches the
    // staged buffer.
    int par = 0;
    if (gt == 0) cs[1 + 2 * gid] = atomicAdd(&cs[0], 1u);
    group_bar(1 + gid, NTG);
    for (;;) {
        const int k = (int)cs[1 + 2 * gid + par];
        if (k >= K) break;
        ACA_CHECK(k >= 0, k, gid);
        ACA_TRACE(1, k);
        const int b = k % NBUF;
        unsigned long long* S = Sb + b * NSLOTP;
        // Tile k is phase u = k / NBUF of bar[b]. A fast group may claim tile k while tile k - NBUF
        // (the same buffer) is still being processed by a slow group, i.e. before phase u is even
        // armed; a parity wait then would alias phase u - 1 (already complete). So wait until
        // phase u is armed, then for its completion.
        {
            const unsigned int use = (unsigned int)(k / NBUF);
            while (armed[b] <= use) __nanosleep(64);
            mbar_wait(&bar[b], use & 1u);
        }
        const Org o = org_load(k);
        const bool fast = o.full && vec_ok;
        bool patched = !fast && o.valid;   // threads wrote words into the buffer: barrier before use
        if (fast) {   // the words the bulk copies left out: x-halo columns, unsafe face rows
            patched = !x_tma(o);
            if (!x_tma(o)) {
                for (int h = gt; h < 2 * NROWS; h += NTG) {
                    const int row = h >> 1, lx = (h & 1) ? TX : -1, ly = row % TY, lz = row / TY;
                    S[slot(lx, ly, lz)] = ld_word_t<true>(P, o.x0 + lx, o.y0 + ly, o.z0 + lz);
                }
                if (MOORE && gt < 4) {   // the four corner cells (diagonal neighbours)
                    const int lx = (gt & 1) ? TX : -1, ly = (gt & 2) ? TY : -1;
                    S[slot(lx, ly, 0)] = ld_word_t<true>(P, o.x0 + lx, o.y0 + ly, 0);
                }
            }
            // face rows of a category (2-D: y-; y+. 3-D: z-, z+ (TY rows each); y-, y+ (TZ rows each))
            // whose bulk copy was unsafe: by threads
            const int ncat = NDIM == 2 ? 2 : 4;
            for (int c = 0; c < ncat; ++c) {
                const bool zface = NDIM == 3 && c < 2, lo = (c & 1) == 0;
                if (face_ok(o, zface, lo)) continue;
                patched = true;
                const int f0 = NDIM == 2 ? c : (c < 2 ? c * TY : 2 * TY + (c - 2) * TZ);
                const int nf = NDIM == 2 ? 1 : (c < 2 ? TY : TZ);
                for (int h = gt; h < nf * (TX + 2); h += NTG) {
                    int ly, lz;
                    face_coords(f0 + h / (TX + 2), ly, lz);
                    const int lx = h % (TX + 2) - 1;
                    S[slot(lx, ly, lz)] = ld_word_t<true>(P, o.x0 + lx, o.y0 + ly, o.z0 + lz);
                }
            }
        } else if (o.valid) {   // ragged or odd-width tile: the whole slot set by threads
            for (int i = gt; i < NSLOT; i += NTG) {
                const int lx = i % SX - 2, ly = (i / SX) % SY - 1, lz = (NDIM == 3) ? i / SXY - 1 : 0;
                if (lx < -1 || lx > TX) continue;
                const int out = (lx < 0 || lx >= TX) + (ly < 0 || ly >= TY) + ((NDIM == 3) && (lz < 0 || lz >= TZ));
                if (MOORE || out <= 1) S[i] = ld_word(P, o.x0 + lx, o.y0 + ly, o.z0 + lz);
            }
        }
        if (patched) group_bar(1 + gid, NTG);
        ACA_TRACE(2, ((unsigned long long)o.x0 << 32) | (unsigned)o.y0);

        if (o.valid) {
            unsigned int rounds;
#ifdef ACA_ABL_CLS_EARLYONLY
            if (true) {
#else
            if (!CLS || o.early) {
#endif
                rounds = o.full ? tile_rounds<NDIM, TX, TY, TZ, NTG, true, EARLY, MOORE, GEN>(P, S, q, wg, thr_a, thr, thm, tab,
                                                                                             o.x0, o.y0, o.z0, wlim, st)
                                : tile_rounds<NDIM, TX, TY, TZ, NTG, false, EARLY, MOORE, GEN>(P, S, q, wg, thr_a, thr, thm, tab,
                                                                                              o.x0, o.y0, o.z0, wlim, st);
            } else {
                rounds = o.full ? tile_rounds<NDIM, TX, TY, TZ, NTG, true, false, MOORE, GEN>(P, S, q, wg, thr_a, thr, thm, tab,
                                                                                             o.x0, o.y0, o.z0, wlim, st)
                                : tile_rounds<NDIM, TX, TY, TZ, NTG, false, false, MOORE, GEN>(P, S, q, wg, thr_a, thr, thm, tab,
                                                                                              o.x0, o.y0, o.z0, wlim, st);
            }
            if (CLS && gt == 0) atomicAdd(&cs[o.early ? 30 : 31], 1u);   // CLS: visits per path
            unsigned long long c0 = 0, c1 = 0;   // CLS: per-lane class counters of this visit (per-cell count)
            rounds_max = rounds > rounds_max ? rounds : rounds_max;
            tot.fold(st);
            if (fast) {
                // Per-warp write-back: a warp's own cells (tile-linear [wg CPW, (wg + 1) CPW))
                // are final once its round loop ends, so each warp stores its rows while the
                // others may still be firing.
                const int wb0 = wg * CPW;
                const unsigned long long wT = lagw[1];   // T (termination counts cells below it)
                unsigned long long wm = ~0ull;
                // the lag minimum only when a lag window is set: two copies of the loop in the a10
                // kernels (c5 +1.1 %), the runtime test in the plain ones (c3: the copies cost
                // 0.4-1.2 %; r02g A/B)
                const bool lag = P.lag_q != 0;
                auto write_back = [&](auto LAGC) {
                    for (int idx = lane; idx < CPW / 2; idx += 32) {
                        const int oo = wb0 + 2 * idx;
                        const int lx = oo % TX, ly = (oo / TX) % TY, lz = oo / (TX * TY);
                        const size_t gi = NDIM == 2 ? (size_t)(o.y0 + ly) * g.nx + o.x0 + lx
                                                    : ((size_t)(o.z0 + lz) * g.ny + (o.y0 + ly)) * g.nx + o.x0 + lx;
                        const ulonglong2 v = lds128v(&S[slot(lx, ly, lz)]);
                        if constexpr (BMC) {   // spin bits of the row's even / odd columns
                            const unsigned int be = __ballot_sync(0xffffffffu, (unsigned int)v.x & 1u);
                            const unsigned int bo = __ballot_sync(0xffffffffu, (unsigned int)v.y & 1u);
                            if (lane == 0) {
                                unsigned int* bm = cbm + (gid * 2 + par) * CBMW;
                                bm[ly + 1] = be;
                                bm[TY + 2 + ly + 1] = bo;
                            }
                        } else if constexpr (CLS) {
                            cls_pair<NDIM, SX, SXY>(S, slot(lx, ly, lz), v, c0, c1);
                        }
                        ACA_CHECK(gi + 1 < (size_t)g.nx * g.ny * g.nz, gi, oo);
                        *reinterpret_cast<ulonglong2*>(P.words + gi) = v;
                        active += (v.x < wT) + (v.y < wT);
                        if constexpr (EARLY != 0) {
                            if constexpr (decltype(LAGC)::value) wm = min(wm, min(v.x, v.y));
                        } else {
                            if (lag) wm = min(wm, min(v.x, v.y));
                        }
                        if (P.push_lo) {
                            const int a = NDIM == 2 ? o.y0 + ly : o.z0 + lz, n = NDIM == 2 ? g.ny : g.nz;
                            if (a == 0 || a == n - 1) {
                                const size_t f = NDIM == 2 ? (size_t)(o.x0 + lx) : (size_t)(o.y0 + ly) * g.nx + o.x0 + lx;
                                *reinterpret_cast<ulonglong2*>((a == 0 ? P.push_lo : P.push_hi) + f) = v;
                                if (a == 0 && n == 1) *reinterpret_cast<ulonglong2*>(P.push_hi + f) = v;
                            }
                        }
                    }
                };
                if (EARLY == 0 || lag) write_back(BoolC<true>{});
                else write_back(BoolC<false>{});
                if (P.lag_q) atomicMin(&lagw[0], wm);
                if constexpr (BMC) {   // the x-halo spins of the warp's rows; the face rows
                    unsigned int* bm = cbm + (gid * 2 + par) * CBMW;
                    constexpr int RPWB = CPW / TX;
                    const int r0 = wb0 / TX;
                    if (lane < RPWB) {
                        const int row = r0 + lane;
                        const unsigned int hb = (unsigned int)(S[slot(-1, row, 0)] & 1ull) |
                                                ((unsigned int)(S[slot(TX, row, 0)] & 1ull) << 1);
                        reinterpret_cast<unsigned char*>(bm + 2 * (TY + 2))[row] = (unsigned char)hb;
                    }
#pragma unroll
                    for (int f = 0; f < 2; ++f) {
                        if ((f == 0 && wg == 0) || (f == 1 && wg == NWG - 1)) {
                            const int ly = f == 0 ? -1 : TY;
                            const ulonglong2 v = lds128v(&S[slot(2 * lane, ly, 0)]);
                            const unsigned int be = __ballot_sync(0xffffffffu, (unsigned int)v.x & 1u);
                            const unsigned int bo = __ballot_sync(0xffffffffu, (unsigned int)v.y & 1u);
                            if (lane == 0) {
                                bm[ly + 1] = be;
                                bm[TY + 2 + ly + 1] = bo;
                            }
                        }
                    }
                }
            } else {
                group_bar(1 + gid, NTG);   // other warps' cells are read below
                for (int oo = gt; oo < NCELL; oo += NTG) {
                    const int lx = oo % TX, ly = (oo / TX) % TY, lz = oo / (TX * TY);
                    const int gx = o.x0 + lx, gy = o.y0 + ly, gz = o.z0 + lz;
                    if (gx < g.nx && gy < g.ny && (NDIM == 2 || gz < g.nz)) {
                        const size_t gi = NDIM == 2 ? (size_t)gy * g.nx + gx : ((size_t)gz * g.ny + gy) * g.nx + gx;
                        const unsigned long long w = S[slot(lx, ly, lz)];
                        if constexpr (CLS) cls_one<NDIM, SX, SXY>(S, slot(lx, ly, lz), w, c0, c1);
                        P.words[gi] = w;
                        push_word(P, gx, gy, gz, w);
                        active += w < lagw[1];
                        if (P.lag_q) atomicMin(&lagw[0], w);
                    }
                }
            }
            if constexpr (CLS) {
                if (!(BMC && fast)) cls_flush_warp<NBIN>(c0, c1, ghist + (gid * 2 + par) * 16, lane);
            }
        }
        ACA_TRACE(6, k);
        if constexpr (BMC) {
            // The classes of the group's previous visit (bitmap set par ^ 1, final since that
            // visit's closing barrier) are counted now, by every warp for its own rows, in the
            // time it would otherwise wait at this visit's closing barrier; the group's thread 0
            // writes them to HBM after that barrier. This visit's set is marked for the next one.
            unsigned int* pb = cbm + (gid * 2 + (par ^ 1)) * CBMW;
            if (pb[2 * (TY + 2) + (TY + 3) / 4 + 16] != ~0u) cls_count_rows<TY, NCELL / NWG / TX>(pb, wg * (NCELL / NWG / TX), lane);
            if (gt == 0)
                cbm[(gid * 2 + par) * CBMW + 2 * (TY + 2) + (TY + 3) / 4 + 16] =
                    (fast && o.valid) ? (unsigned int)tile_index(o) : ~0u;
        }
        // refill the buffer with tile k + NBUF: armed before the barrier (the arrive does not
        // touch the buffer), copied after it by every thread of the group (at most a row each)
        if (gt == 0) {
            if (k + NBUF < K) arm(k + NBUF, b);
            cs[1 + 2 * gid + (par ^ 1)] = atomicAdd(&cs[0], 1u);   // the group's next tile
        }
        group_bar(1 + gid, NTG);   // the buffer is free
        ACA_TRACE(7, k);
        if constexpr (CLS) {   // the tile's class histogram of this visit -> HBM (and zeroed for reuse)
            if (BMC && gt == 0) {   // the previous visit's deferred histogram (counted before this barrier)
                unsigned int* dh = cbm + (gid * 2 + (par ^ 1)) * CBMW + 2 * (TY + 2) + (TY + 3) / 4;
                if (dh[16] != ~0u) {
                    uint4* hp = reinterpret_cast<uint4*>(P.tile_hist + 16 * (size_t)dh[16]);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        hp[j] = make_uint4(dh[4 * j], dh[4 * j + 1], dh[4 * j + 2], dh[4 * j + 3]);
                        dh[4 * j] = dh[4 * j + 1] = dh[4 * j + 2] = dh[4 * j + 3] = 0u;
                    }
                    dh[16] = ~0u;
                }
            }
            if (BMC && fast && o.valid) {
                // counted during the group's next visit (or after the loop)
            } else if (gt == 0 && o.valid) {
                unsigned int* gh = ghist + (gid * 2 + par) * 16;
                uint4* hp = reinterpret_cast<uint4*>(P.tile_hist + 16 * tile_index(o));
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    hp[j] = make_uint4(gh[4 * j], gh[4 * j + 1], gh[4 * j + 2], gh[4 * j + 3]);
                    gh[4 * j] = gh[4 * j + 1] = gh[4 * j + 2] = gh[4 * j + 3] = 0u;
                }
            }
        }
        par ^= 1;
        if (k + NBUF < K) copy_rows(k + NBUF, gt, NTG);
    }
    ACA_TRACE(8, 0);
    if constexpr (BMC) {   // the group's last visit: count its set (par ^ 1) and write it
        unsigned int* pb = cbm + (gid * 2 + (par ^ 1)) * CBMW;
        unsigned int* dh = pb + 2 * (TY + 2) + (TY + 3) / 4;
        if (dh[16] != ~0u) cls_count_rows<TY, NCELL / NWG / TX>(pb, wg * (NCELL / NWG / TX), lane);
        group_bar(1 + gid, NTG);
        if (gt == 0 && dh[16] != ~0u) {
            uint4* hp = reinterpret_cast<uint4*>(P.tile_hist + 16 * (size_t)dh[16]);
#pragma unroll
            for (int j = 0; j < 4; ++j) hp[j] = make_uint4(dh[4 * j], dh[4 * j + 1], dh[4 * j + 2], dh[4 * j + 3]);
        }
    }
    __syncthreads();
    if (P.lag_q && tid == 0 && lagw[0] != ~0ull) atomicMin(&P.ctl->wmin[P.phase > 0 ? 1 : 0], lagw[0]);
    const unsigned long long s_act = block_sum<NT>((unsigned long long)active, red);
    tot.fold(st);
    const unsigned long long s_fir = block_sum<NT>(tot.fired, red);
    const unsigned long long s_flp = block_sum<NT>(tot.flips, red);
    const unsigned long long s_tst = block_sum<NT>(tot.tested, red);
    const unsigned long long s_hsh = block_sum<NT>(st.hacc, red);
    if constexpr (CLS) {
        if (tid == 0 && cs[30]) atomicAdd(&P.ctl->visits_early, (unsigned long long)cs[30]);
        if (tid == 0 && cs[31]) atomicAdd(&P.ctl->visits_plain, (unsigned long long)cs[31]);
    }
    if (tid == 0) finish_launch(P.ctl, s_act, s_fir, s_flp, s_tst, s_hsh, rounds_max, P.phase, P.lag_q, g.TSH);
}
