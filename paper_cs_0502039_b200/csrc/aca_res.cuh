// aca_res.cuh — resident-tile persistent kernel for small 2-D lattices (config 2); included by
// aca_kernels.cuh inside namespace aca.
//
// A lattice whose 64 x 64 tiles fit in the shared memory of the GPU's SMs (two per colour per
// CTA) need not stream its state through HBM / L2 every sweep, nor pay a kernel launch, a table
// load and a staging per tile visit: one cooperative launch runs the whole run_until. Every CTA
// keeps its tiles (its share of each checkerboard colour) in shared memory; a sweep is the two
// colours in turn (fig:amcgen's outer round), separated by grid barriers. A
// tile's visit reloads its one-cell halo from global memory (the neighbours' boundary words,
// written back at the end of their own visits, before the barrier), runs the in-tile rounds of
// the production kernel (tile_rounds, fig:s1c1pe PAPER.md:682-715), and writes back its four
// boundary lines; the interior stays in shared memory until the run ends. The schedule is the
// checkerboard one of tile_grp_kernel, so the trajectory is the same unique one.
// Termination: after each sweep every CTA has added the active cells (t < T) of its tiles to
// ctl->res_act[sweep % 3]; after the barrier all CTAs read the total and stop at 0.

__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// grid-wide barrier of a cooperative launch (every CTA co-resident)
__device__ __forceinline__ void res_grid_sync(Ctl* ctl) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int gen = ld_acquire_u32(&ctl->bar_gen);
        __threadfence();
        if (atomicAdd(&ctl->bar_count, 1u) == gridDim.x - 1) {
            ctl->bar_count = 0u;
            __threadfence();
            atomicAdd(&ctl->bar_gen, 1u);
        } else {
            while (ld_acquire_u32(&ctl->bar_gen) == gen) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

__host__ __device__ constexpr int res_tiles_max() { return 4; }   // resident tiles per CTA (2 per colour)
__host__ __device__ constexpr size_t res_smem_bytes(int nt) {
    return ((size_t)res_tiles_max() * grp_slots(2, 64, 64, 1) + 16 + 112 + 256 + 128 + nt / 32) * 8 +
           (((size_t)(nt / 32) * tile_queue_per_warp(4096 / (nt / 32), false) * 2 + 15) & ~(size_t)15);
}

template <int NT>
__global__ void __launch_bounds__(NT, 1) res_kernel(const __grid_constant__ KParams P) {
    constexpr int NDIM = 2, TX = 64, TY = 64, TZ = 1;
    constexpr int SX = TX + 4;
    constexpr int NSLOTP = grp_slots(2, TX, TY, TZ);
    constexpr int NW = NT / 32;
    constexpr int CPW = TX * TY / NW;
    constexpr int QW = tile_queue_per_warp(CPW, false);
    constexpr int HALF = res_tiles_max() / 2;
    if (*(volatile unsigned int*)&P.ctl->done) return;

    extern __shared__ __align__(128) unsigned long long smem[];
    unsigned long long* Sb = smem;                                    // res_tiles_max() x NSLOTP
    unsigned long long* thr = Sb + res_tiles_max() * NSLOTP;          // 16
    unsigned long long* thm = thr + 16;                               // 112 (unused: no a10)
    unsigned long long* Lt = thm + 112;                               // 256
    unsigned int* Rt = (unsigned int*)(Lt + 256);                     // 256 u32
    unsigned long long* red = Lt + 256 + 128;                         // NW
    unsigned short* Q = (unsigned short*)(red + NW);                  // NW x QW

    const Geo& g = P.g;
    const int tid = threadIdx.x, warp = tid >> 5;
    if (tid < 16) thr[tid] = tid < 14 ? P.thr[tid] : 0ull;
    for (int i = tid; i < 112; i += NT) thm[i] = ~0ull;
    for (int i = tid; i < 256; i += NT) {
        Lt[i] = P.lr[2 * i];
        Rt[i] = (unsigned int)P.lr[2 * i + 1];
    }
    const NlogSmem tab{smem_u32(Lt), smem_u32(Rt)};
    const uint32_t thr_a = smem_u32(thr);
    unsigned short* q = Q + warp * QW;
    const unsigned long long wlim = *(volatile unsigned long long*)&P.ctl->wlim;
    auto slot = [](int lx, int ly) { return (ly + 1) * SX + lx + 2; };

    // this CTA's tiles: colour c, item blockIdx.x + j gridDim.x of the colour's list (as in
    // tile_grp_kernel: item -> tile row, column pair), in buffer c HALF + j
    const int hx = (P.tiles_x + 1) >> 1;
    const int nitems = hx * P.tiles_y;
    auto org = [&](int c, int j, int& x0, int& y0) -> bool {
        const int it = (int)blockIdx.x + j * (int)gridDim.x;
        if (it >= nitems) return false;
        const int ty = it / hx;
        const int tx = 2 * (it % hx) + ((ty + c) & 1);
        if (tx >= P.tiles_x) return false;
        x0 = tx * TX;
        y0 = ty * TY;
        return true;
    };
    // stage every resident tile (own cells and halo)
    for (int c = 0; c < 2; ++c)
        for (int j = 0; j < HALF; ++j) {
            int x0, y0;
            if (!org(c, j, x0, y0)) continue;
            unsigned long long* S = Sb + (c * HALF + j) * NSLOTP;
            for (int i = tid; i < (TX + 2) * (TY + 2); i += NT) {
                const int lx = i % (TX + 2) - 1, ly = i / (TX + 2) - 1;
                if ((lx < 0 || lx >= TX) && (ly < 0 || ly >= TY)) continue;   // corners: unused
                S[slot(lx, ly)] = ld_word_t<true>(P, x0 + lx, y0 + ly, 0);
            }
        }
    __syncthreads();

    TileStats st;
    TileTotals tot;
    unsigned int rounds_sum = 0;
    unsigned long long sweeps = 0;
    for (unsigned long long sw = 0;; ++sw) {
        unsigned long long act = 0;   // thread-local: active own cells of this CTA's tiles
        for (int c = 0; c < 2; ++c) {
            unsigned int rmax = 0;
            for (int j = 0; j < HALF; ++j) {
                int x0, y0;
                if (!org(c, j, x0, y0)) continue;
                unsigned long long* S = Sb + (c * HALF + j) * NSLOTP;
                if (sw > 0 || c > 0) {   // the neighbours' boundary words of this sweep
                    for (int i = tid; i < 4 * TX; i += NT) {
                        const int side = i / TX, k = i % TX;
                        const int lx = side == 0 ? -1 : side == 1 ? TX : k;
                        const int ly = side == 2 ? -1 : side == 3 ? TY : k;
                        S[slot(lx, ly)] = ld_word_t<true>(P, x0 + lx, y0 + ly, 0);
                    }
                    __syncthreads();
                }
                const unsigned int r = tile_rounds<NDIM, TX, TY, TZ, NT, true, false, false, false>(
                    P, S, q, warp, thr_a, thr, thm, tab, x0, y0, 0, wlim, st);
                rmax = r > rmax ? r : rmax;
                tot.fold(st);
                __syncthreads();   // every warp's rows are final for this visit
                // the four boundary lines -> global (read by the neighbours after the barrier)
                for (int i = tid; i < 4 * TX; i += NT) {
                    const int side = i / TX, k = i % TX;
                    const int lx = side == 0 ? 0 : side == 1 ? TX - 1 : k;
                    const int ly = side == 2 ? 0 : side == 3 ? TY - 1 : k;
                    P.words[(size_t)(y0 + ly) * g.nx + x0 + lx] = S[slot(lx, ly)];
                }
                for (int i = tid; i < TX * TY; i += NT) act += S[slot(i % TX, i / TX)] < wlim;
            }
            rounds_sum += rmax;
            if (c == 0) {
                res_grid_sync(P.ctl);
                // every CTA has read res_act of the previous sweep: clear it for the sweep after next
                if (blockIdx.x == 0 && tid == 0 && sw > 0) P.ctl->res_act[(sw - 1) % 3] = 0ull;
            }
        }
        const unsigned long long a = block_sum<NT>(act, red);
        if (tid == 0 && a) atomicAdd(&P.ctl->res_act[sw % 3], a);
        res_grid_sync(P.ctl);
        ++sweeps;
        __shared__ int stop;
        if (tid == 0) {
            const unsigned long long tot_act = *(volatile unsigned long long*)&P.ctl->res_act[sw % 3];
            stop = tot_act == 0ull || *(volatile unsigned int*)&P.ctl->overflow;
        }
        __syncthreads();
        if (stop) break;
    }
    // the interiors -> global
    for (int c = 0; c < 2; ++c)
        for (int j = 0; j < HALF; ++j) {
            int x0, y0;
            if (!org(c, j, x0, y0)) continue;
            const unsigned long long* S = Sb + (c * HALF + j) * NSLOTP;
            for (int i = tid; i < TX * TY; i += NT)
                P.words[(size_t)(y0 + i / TX) * g.nx + x0 + i % TX] = S[slot(i % TX, i / TX)];
        }
    tot.fold(st);
    const unsigned long long s_fir = block_sum<NT>(tot.fired, red);
    const unsigned long long s_flp = block_sum<NT>(tot.flips, red);
    const unsigned long long s_tst = block_sum<NT>(tot.tested, red);
    const unsigned long long s_hsh = block_sum<NT>(st.hacc, red);
    if (tid == 0) {
        if (s_fir) atomicAdd(&P.ctl->fired, s_fir);
        if (s_flp) atomicAdd(&P.ctl->flips, s_flp);
        if (s_tst) atomicAdd(&P.ctl->tested, s_tst);
        if (s_hsh) atomicAdd(&P.ctl->hash, s_hsh);
        if (blockIdx.x == 0) {
            P.ctl->launches += sweeps;
            P.ctl->inner_rounds += rounds_sum;
            P.ctl->active_last = 0ull;
            P.ctl->res_act[0] = P.ctl->res_act[1] = P.ctl->res_act[2] = 0ull;
            P.ctl->done = 1u;
        }
    }
}
