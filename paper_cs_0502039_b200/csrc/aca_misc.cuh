// aca_misc.cuh — the whole-lattice kernel and the one-pass kernels (init, frames, pack,
// repack, gather, unpack, statistics); included by aca_kernels.cuh inside namespace aca.

// ------------------------------------------------------------ whole-lattice kernel
// One CTA holds the entire (small) lattice in shared memory with true periodic addressing
// and runs rounds until no cell has t < T: the whole run_until in one launch. This is the
// configuration-1 "one cell per PE" arrangement (fig:s1c1pe) with the
// 2^14-PE Connection Machine replaced by one CTA.
template <int NT, bool SYNC>
__global__ void __launch_bounds__(NT) whole_kernel(const KParams P) {
    const Geo& g = P.g;
    if (*(volatile unsigned int*)&P.ctl->done) return;
    extern __shared__ __align__(128) unsigned long long smem[];
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
            // P6: (t, c) order with the explicit id order of the periodic neighbours
            bool ok = lex_lt(w, a, g.TSH, x == 0) && lex_lt(w, b, g.TSH, x < g.nx - 1) &&
                      lex_lt(w, c2, g.TSH, y == 0) && lex_lt(w, d2, g.TSH, y < g.ny - 1);
            uint32_t ones = (uint32_t)(a & 1ull) + (uint32_t)(b & 1ull) + (uint32_t)(c2 & 1ull) + (uint32_t)(d2 & 1ull);
            if (P.life) {   // Moore neighbourhood, explicit (t, c) order
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
                ok = ok && lex_lt(w, e, g.TSH, z == 0) && lex_lt(w, f, g.TSH, z < g.nz - 1);
                ones += (uint32_t)(e & 1ull) + (uint32_t)(f & 1ull);
            }
            if (!ok) continue;
            const FireOut o = fire(w, ones, P.life ? 8 : Z, (unsigned long long)i, g, thr, NlogLR{lr}, P.rk, P.inv_lambda,
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
            const unsigned long long c = cbase + x;
            const u32x4 r = philox4x32_10_rk(0u, (uint32_t)c, (uint32_t)(c >> 32), 1u, K.rk);
            const unsigned long long sb = ((unsigned long long)r.x < thr_init) ? 0ull : 1ull;
            const unsigned long long t0 = delta_cell_t(c, K.rk, r.y, r.z, NlogLR{lr}, ACA_LN2_Q48, inv_lambda, tie_bits, law);
            words[(size_t)row * nx + x] = w_pack(t0, 0ull, sb, g);
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
                            Geo g, unsigned long long n) {
    if (spins && !times && !counters) {   // spins only: the (t, n) fields are unchanged
        for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
             i += (unsigned long long)gridDim.x * blockDim.x)
            words[i] = (words[i] & ~1ull) | (spins[i] > 0 ? 1ull : 0ull);
        return;
    }
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long w = words[i];
        const unsigned long long t = times ? times[i] : w_time(w, g);
        const unsigned long long k = counters ? counters[i] : w_count(w, g);
        const unsigned long long sb = spins ? (spins[i] > 0 ? 1ull : 0ull) : (w & 1ull);
        words[i] = w_pack(t, k, sb, g);
    }
}

// Change the (t, n) split of the words in place (from layout a to layout b).
__global__ void repack_kernel(unsigned long long* __restrict__ words, Geo a, Geo b, unsigned long long n) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long w = words[i];
        words[i] = w_pack(w_time(w, a), w_count(w, a), w & 1ull, b);
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


// a10 per-tile class bookkeeping: the BKL class histogram (P4 index of (s, Sigma),
// PAPER.md:1039-1045) of every tile of a shard from the current state, into P.tile_hist (16 u32
// per tile, tile index (tz tiles_y + ty) tiles_x + tx as in tile_grp_kernel). Run when the state
// is set from outside (create, reset, set_state/set_spins) and by aca_get_tile_classes with
// refresh = 1; during runs the tile kernel recounts a tile at every visit. One CTA per tile.
template <int NT>
__global__ void __launch_bounds__(NT) class_refresh_kernel(const KParams P, int TX, int TY, int TZ) {
    __shared__ unsigned int h[16];
    const Geo& g = P.g;
    if (threadIdx.x < 16) h[threadIdx.x] = 0u;
    __syncthreads();
    const int t = blockIdx.x;
    const int tx = t % P.tiles_x, ty = (t / P.tiles_x) % P.tiles_y, tz = t / (P.tiles_x * P.tiles_y);
    const uint32_t Z = 2 * g.ndim;
    for (int i = threadIdx.x; i < TX * TY * TZ; i += NT) {
        const int x = tx * TX + i % TX, y = ty * TY + (i / TX) % TY, z = tz * TZ + i / (TX * TY);
        if (x >= g.nx || y >= g.ny || (g.ndim == 3 && z >= g.nz)) continue;
        const unsigned long long w = *word_ptr_t<false>(P, x, y, z);
        uint32_t o = (uint32_t)(*word_ptr_t<false>(P, x - 1, y, z) & 1ull) + (uint32_t)(*word_ptr_t<false>(P, x + 1, y, z) & 1ull) +
                     (uint32_t)(*word_ptr_t<false>(P, x, y - 1, z) & 1ull) + (uint32_t)(*word_ptr_t<false>(P, x, y + 1, z) & 1ull);
        if (g.ndim == 3)
            o += (uint32_t)(*word_ptr_t<false>(P, x, y, z - 1) & 1ull) + (uint32_t)(*word_ptr_t<false>(P, x, y, z + 1) & 1ull);
        atomicAdd(&h[o + (Z + 1) * (uint32_t)(w & 1ull)], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 16) P.tile_hist[16 * (size_t)t + threadIdx.x] = h[threadIdx.x];
}
