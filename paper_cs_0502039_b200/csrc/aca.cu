// aca.cu — C-ABI runtime of the B200 path (include/aca.h). Host side: validation, P4 table,
// device allocation, the packed-word layout, shard/halo bookkeeping, the outer-round loop
// (CUDA-graph replay of K launches, device-side termination, two batches in flight),
// statistics and getters. Every step of the method runs in the kernels of aca_kernels.cuh;
// nothing here computes a trajectory.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <curand_kernel.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <thread>
#include <chrono>

#include "../../include/aca.h"
#include "aca_kernels.cuh"
#include "aca_eff.cuh"
#include "aca_agg.cuh"
#include "aca_qnbr.cuh"
#include "nlog_tables.cuh"

using namespace aca;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(ACA_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_),    \
                        __FILE__, __LINE__);                                                  \
    } while (0)

// ---------------------------------------------------------------- NCCL (resolved at runtime)
// The library never links NCCL; when world > 1 it resolves the symbols of the libnccl that
// the process already loaded (torch's), so the halo exchange uses the same NCCL as the
// process group that distributed the ncclUniqueId.
typedef struct { char internal[128]; } ncclUniqueId_t;
typedef void* ncclComm_t;
typedef int (*ncclCommInitRank_fn)(ncclComm_t*, int, ncclUniqueId_t, int);
typedef int (*ncclCommDestroy_fn)(ncclComm_t);
typedef int (*ncclSend_fn)(const void*, size_t, int, int, ncclComm_t, cudaStream_t);
typedef int (*ncclRecv_fn)(void*, size_t, int, int, ncclComm_t, cudaStream_t);
typedef int (*ncclGroup_fn)(void);
typedef int (*ncclAllReduce_fn)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t);
typedef int (*ncclGetUniqueId_fn)(ncclUniqueId_t*);
struct NcclApi {
    ncclCommInitRank_fn init = nullptr;
    ncclCommDestroy_fn destroy = nullptr;
    ncclSend_fn send = nullptr;
    ncclRecv_fn recv = nullptr;
    ncclGroup_fn gstart = nullptr, gend = nullptr;
    ncclAllReduce_fn allreduce = nullptr;
    ncclGetUniqueId_fn uid = nullptr;
    bool ok = false;
};
NcclApi& nccl() {
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* h = dlopen(nullptr, RTLD_NOW);
        auto sym = [&](const char* n) -> void* {
            void* p = h ? dlsym(h, n) : nullptr;
            if (!p) {
                static void* lib = nullptr;
                if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
                if (lib) p = dlsym(lib, n);
            }
            return p;
        };
        api.init = (ncclCommInitRank_fn)sym("ncclCommInitRank");
        api.destroy = (ncclCommDestroy_fn)sym("ncclCommDestroy");
        api.send = (ncclSend_fn)sym("ncclSend");
        api.recv = (ncclRecv_fn)sym("ncclRecv");
        api.gstart = (ncclGroup_fn)sym("ncclGroupStart");
        api.gend = (ncclGroup_fn)sym("ncclGroupEnd");
        api.allreduce = (ncclAllReduce_fn)sym("ncclAllReduce");
        api.uid = (ncclGetUniqueId_fn)sym("ncclGetUniqueId");
        api.ok = api.init && api.destroy && api.send && api.recv && api.gstart && api.gend && api.allreduce;
    }
    return api;
}
constexpr int NCCL_UINT8 = 1, NCCL_UINT64 = 5, NCCL_SUM = 0;

struct Shard {
    Geo g{};
    unsigned long long* words = nullptr;
    unsigned long long* halo_lo = nullptr;  // 1 row (2-D) / plane (3-D)
    unsigned long long* halo_hi = nullptr;
    unsigned long long* push_lo = nullptr;  // push mode: the lower neighbour's halo_hi
    unsigned long long* push_hi = nullptr;  // ... and the upper neighbour's halo_lo
    unsigned long long* stats_lo = nullptr; // multi-process: the halos as they were at the end of the last run
    unsigned long long* stats_hi = nullptr; //   (the bond term of the statistics reads these)
    Ctl* ctl = nullptr;
    size_t n = 0;          // owned cells
    size_t face = 0;       // cells of one row / plane of the sharded axis
    int tiles_x = 1, tiles_y = 1, tiles_z = 1;
    unsigned int* tile_hist = nullptr;      // a10 class bookkeeping: 16 u32 per tile (class_book)
    CUtensorMap tmap{};                     // TMA box of one tile over `words` (box_ok = 1 when encoded)
    int box_ok = 0;
};

}  // namespace

struct aca_sim {
    int ndim = 2;
    int64_t dims[3] = {1, 1, 1};
    int64_t N = 0;          // whole lattice
    double lambda = 1, beta = 0, J = 1, h = 0;
    int rule = 0;
    uint64_t seed = 0;
    aca_options opt{};
    int device = 0;
    int NB = 1, TB = 1;            // packed word: counter bits, time bits (+1 spin bit)
    uint64_t t_hi = 0;             // exclusive upper bound of every stored time (Q32)
    bool sync_debug = false;       // ACA_SYNC_DEBUG=1: synchronise after every tile launch
    unsigned long long lag_q = 0;  // bounded lag (aca_options.lag / lambda) in Q32; 0 = off
    unsigned long long* h_trace = nullptr;   // ACA_TRACE_FROM=n (debug builds): host-mapped stage trace
    unsigned long long* h_dbg = nullptr;     // ACA_SYNC_DEBUG (debug builds): host-mapped failed-check record
    long long trace_from = -1;
    unsigned long long inv_lambda = 1ull << 32;
    unsigned long long thr[14] = {};
    unsigned long long thm[98] = {};   // a10 early-rejection table (see commit_loop)
    bool cls = false;                  // a10 per-tile class bookkeeping (aca_options.class_book)
    // resident-tile kernel (small 2-D lattices): the whole run_until in one cooperative launch
    bool res_ok = false;
    int res_grid = 0;
    int res_nt = 512;                  // threads per CTA (one tile at a time)
    void* res_fn = nullptr;
    size_t res_smem = 0;
    bool cls_stale = true;             // the tile histograms must be recounted before the next run
    long long cls_lim = -1;            // early path iff sum_k |Gamma_k| floor(p_k 2^16) <= cls_lim
    int bulk = 1;
    unsigned long long thr_init = 0;
    unsigned long long max_delta = 0;
    uint64_t T_last = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    // asynchronous spin I/O (aca_stage_spins / aca_set_spins_staged / aca_get_spins_async)
    cudaStream_t cstream = nullptr;           // copy stream
    int8_t* stage_in[2] = {nullptr, nullptr};
    int8_t* stage_out[2] = {nullptr, nullptr};
    cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_pack[2] = {nullptr, nullptr};
    cudaEvent_t ev_unp[2] = {nullptr, nullptr}, ev_d2h[2] = {nullptr, nullptr};
    int out_slot = 0;
    unsigned long long* d_lr = nullptr;
    std::vector<Shard> shards;
    int G = 1;                     // shards on this device
    int rank = 0, world = 1;
    bool use_nccl = false;         // nccl_id given: halos travel by NCCL (world >= 1; world 1 = self)
    ncclComm_t comm = nullptr;
    int tile[3] = {64, 64, 1};
    int rounds = 8;
    int K = 16;
    bool whole = false;
    bool sync = false;
    bool phased = false;           // checkerboard sweeps (two launches per outer round)
    bool push = false;             // sharded: boundary rows pushed into the neighbours' halos by the kernel
    bool ipc = false;              // multi-process push mode: halos of the neighbour ranks mapped by CUDA IPC
    bool ipc_ready = false;        // aca_ipc_import done
    unsigned long long* d_slot = nullptr;              // this rank's {epoch, active, snapshot epoch} (exported)
    bool snap_valid = false;       // multi-process: stats_lo/hi hold the neighbours' current boundary rows
    std::vector<unsigned long long*> peer_slot;        // every rank's slot (own = d_slot)
    std::vector<void*> ipc_opened;                     // mappings to close in aca_destroy
    uint64_t epoch = 0;
    size_t smem = 0;
    int persistent_ctas = 0;       // > 0: grid size of the persistent tile kernel
    void* kern = nullptr;          // selected tile/whole kernel
    void* kern_gen = nullptr;      // its instance with the general arrival (launched when !KParams::fast)
    int nthreads = 256;
    cudaGraphExec_t graph = nullptr;
    int graph_rounds = 0;
    bool graph_stale = false;      // same launches, new parameters (reset: the seed's round keys)
    Ctl* h_ctl = nullptr;          // pinned mirror (2 slots per shard)
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t evb[2][3] = {};    // per in-flight batch: start, end of kernels, end of ctl copy
    unsigned long long* d_flag = nullptr;
    unsigned long long* h_flag = nullptr;
    double gpu_seconds = 0;
    double kernel_seconds = 0;
    uint64_t kernel_launches = 0;
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    StatAcc* d_stat = nullptr;
    StatAcc* h_stat = nullptr;
    FrameParams fr{};              // output frames of the current aca_run_frames chunk (nb = 0: off)
    unsigned int* frame_ring = nullptr;
    size_t frame_ring_bytes = 0;
};

namespace {

// ---------------------------------------------------------------- P4 table (host, double)
// Appendix PAPER.md:1691-1701 generalised (docs/PRIMITIVES.md P4).
// zc neighbours: 2 ndim, or |neighbors^q| - 1 for the q-th degree neighbourhood (P12).
void flip_table_z(int zc, double beta, double J, double h, int rule, unsigned long long* out) {
    for (int sb = 0; sb < 2; ++sb) {
        const int s = 2 * sb - 1;
        for (int k = 0; k <= zc; ++k) {
            const int sigma = 2 * k - zc;
            const double dE = 2.0 * (J * (double)s * (double)sigma + h * (double)s);
            const double a = beta * dE;
            double p;
            if (rule == ACA_HEATBATH) {
                if (a >= 0) {
                    const double x = std::exp(-a);
                    p = x / (1.0 + x);
                } else {
                    p = 1.0 / (1.0 + std::exp(a));
                }
            } else {
                p = (dE <= 0) ? 1.0 : std::exp(-a);
            }
            const unsigned long long thr =
                (p == 1.0) ? (1ull << 32) : (unsigned long long)std::floor(p * 4294967296.0);
            out[(sigma + zc) / 2 + (zc + 1) * (s + 1) / 2] = thr;
        }
    }
}

void flip_table(int ndim, double beta, double J, double h, int rule, unsigned long long* out) {
    flip_table_z(2 * ndim, beta, J, h, rule, out);
}

// a10 table: thm[(s*(Z+1) + u)*(Z+1) + k] for a cell with spin bit s, u neighbours that may
// still change before its arrival and k known +1 neighbours. u = 0: the exact threshold.
// u > 0: the largest threshold over the u unknown spins (w0 >= it rejects in every world),
// or "wait" (> 2^32) when early rejection is off or a rejection is less likely than 1/2
// (a Philox draw would mostly be wasted).
void early_table(int ndim, const unsigned long long* thr, bool enabled, unsigned long long* thm) {
    const int Z = 2 * ndim;
    const unsigned long long WAIT = 1ull << 33, CAP = 1ull << 31;
    for (int i = 0; i < 98; ++i) thm[i] = WAIT;
    for (int sb = 0; sb < 2; ++sb)
        for (int u = 0; u <= Z; ++u)
            for (int k = 0; k + u <= Z; ++k) {
                unsigned long long v;
                if (u == 0) {
                    v = thr[k + (Z + 1) * sb];
                } else if (!enabled) {
                    v = WAIT;
                } else {
                    unsigned long long m = 0;
                    for (int j = 0; j <= u; ++j) m = std::max(m, thr[k + j + (Z + 1) * sb]);
                    v = m >= CAP ? WAIT : m;
                }
                thm[(sb * (Z + 1) + u) * (Z + 1) + k] = v;
            }
}

int bits_for(uint64_t v) {
    int b = 0;
    while (v) { ++b; v >>= 1; }
    return b < 1 ? 1 : b;
}

// ---------------------------------------------------------------- kernel registry
// Tile shapes of the production kernel tile_grp_kernel<NDIM, TX, TY, TZ, NTG, NG, NBUF, ...>:
// NG groups of NTG threads per CTA (one CTA per SM) and NBUF tile buffers; (NG_E, NBUF_E) for
// the a10 kernel, whose larger fire queues leave room for fewer buffers. tile_sync_kernel is the
// fig:s1c1pe reference (sync_rounds = 1).
struct TileKey {
    int ndim, tx, ty, tz, ntg;
    void* fn;         // production kernel (the fast arrival only: Poisson law, lambda = 1, no ties/frames)
    void* fn_early;   // with the a10 early-rejection path
    void* fn_gen;     // the same two with the general arrival compiled in (any law, lambda, ties, frames)
    void* fn_early_gen;
    void* fn_life;    // with the Moore neighbourhood (rule 2, 2-D only; nullptr in 3-D)
    void* fn_sync;    // fig:s1c1pe reference kernel
    size_t smem, smem_early, smem_sync;
    int nt, nt_early, nt_sync;
    void* fn_cls;     // a10 path chosen per tile from its class histogram (default shapes only)
    void* fn_cls_gen;
    size_t smem_cls;
};

#define TKG_BASE(ND, TX, TY, TZ, NTG, NG, NBUF, NGE, NBUFE, NTS)                                         \
    {ND, TX, TY, TZ, NTG,                                                                              \
     (void*)tile_grp_kernel<ND, TX, TY, TZ, NTG, NG, NBUF, 0, false, false>,                          \
     (void*)tile_grp_kernel<ND, TX, TY, TZ, NTG, NGE, NBUFE, 1, false, false>,                        \
     (void*)tile_grp_kernel<ND, TX, TY, TZ, NTG, NG, NBUF, 0, false, true>,                           \
     (void*)tile_grp_kernel<ND, TX, TY, TZ, NTG, NGE, NBUFE, 1, false, true>,                         \
     (ND == 2 ? (void*)tile_grp_kernel<ND, TX, TY, TZ, NTG, NG, NBUF, 0, (ND == 2), true> : nullptr), \
     (void*)tile_sync_kernel<ND, TX, TY, TZ, NTS>,                                                     \
     grp_smem_bytes(ND, TX, TY, TZ, NTG, NG, NBUF, false), grp_smem_bytes(ND, TX, TY, TZ, NTG, NGE, NBUFE, true), \
     sync_smem_bytes(ND, TX, TY, TZ, NTS), NTG * NG, NTG * NGE, NTS
#define TKG(ND, TX, TY, TZ, NTG, NG, NBUF, NGE, NBUFE, NTS) \
    TKG_BASE(ND, TX, TY, TZ, NTG, NG, NBUF, NGE, NBUFE, NTS), nullptr, nullptr, 0}
// shapes with the class-bookkeeping instance (the defaults and the few-tile 64x64 group size)
#define TKGC(ND, TX, TY, TZ, NTG, NG, NBUF, NGE, NBUFE, NTS)                                       \
    TKG_BASE(ND, TX, TY, TZ, NTG, NG, NBUF, NGE, NBUFE, NTS),                                      \
        (void*)tile_grp_kernel<ND, TX, TY, TZ, NTG, NGE, NBUFE, 2, false, false>,                  \
        (void*)tile_grp_kernel<ND, TX, TY, TZ, NTG, NGE, NBUFE, 2, false, true>,                   \
        grp_smem_bytes(ND, TX, TY, TZ, NTG, NGE, NBUFE, true, true)}

const TileKey kTiles[] = {
    TKGC(2, 64, 64, 1, 256, 4, 5, 4, 5, 256), TKGC(2, 64, 64, 1, 512, 1, 2, 1, 2, 512),
    TKG(2, 32, 32, 1, 256, 4, 8, 4, 8, 256), TKG(2, 64, 32, 1, 256, 4, 8, 4, 8, 256),
    TKGC(3, 32, 16, 8, 256, 3, 4, 3, 3, 256), TKG(3, 8, 8, 8, 128, 8, 12, 8, 12, 128),
    TKG(3, 16, 16, 16, 256, 3, 4, 3, 3, 256),
};

constexpr int WHOLE_NT = 1024;
size_t whole_smem(int64_t n, bool sync) {
    return (size_t)n * 8 + (512 + 16 + WHOLE_NT / 32) * 8 + (sync ? (size_t)n * 8 : 0);
}

void set_geo_layout(aca_sim* S) {
    for (auto& sh : S->shards) {
        sh.g.NB = S->NB;
        sh.g.TSH = S->NB + 1;
        sh.g.nbmask = (1u << S->NB) - 1u;
    }
}

KParams make_params(const aca_sim* S, const Shard& sh) {
    KParams P{};
    P.g = sh.g;
    P.words = sh.words;
    P.halo_lo = sh.halo_lo;
    P.halo_hi = sh.halo_hi;
    P.push_lo = sh.push_lo;
    P.push_hi = sh.push_hi;
    P.ctl = sh.ctl;
    P.lr = S->d_lr;
    P.key0 = (uint32_t)(S->seed & 0xffffffffu);
    P.key1 = (uint32_t)(S->seed >> 32);
    philox_round_keys(P.key0, P.key1, P.rk);
    P.inv_lambda = S->inv_lambda;
    P.tie_bits = S->opt.tie_bits;
    P.law = S->opt.law;
    P.rounds = S->rounds;
    P.do_hash = S->opt.event_hash;
    P.early = S->opt.early_reject;
    P.bulk = S->bulk;
    P.halo_peer = S->ipc ? 1 : 0;
    P.lag_q = (S->whole || S->sync) ? 0ull : S->lag_q;
    P.dbg_trace = nullptr;
    P.dbg_map = nullptr;
    if (S->h_dbg) {
        void* dp = nullptr;
        if (cudaHostGetDevicePointer(&dp, S->h_dbg, 0) == cudaSuccess) P.dbg_map = (unsigned long long*)dp;
    }
    if (S->h_trace && S->trace_from >= 0 && (long long)S->kernel_launches >= S->trace_from) {
        void* dp = nullptr;
        if (cudaHostGetDevicePointer(&dp, S->h_trace, 0) == cudaSuccess) P.dbg_trace = (unsigned long long*)dp;
    }
    for (int i = 0; i < 98; ++i) P.thm[i] = S->thm[i];
    P.tiles_x = sh.tiles_x;
    P.tiles_y = sh.tiles_y;
    P.tiles_z = sh.tiles_z;
    P.phase = -1;
    P.fr = S->fr;
    P.life = S->rule == ACA_LIFE ? 1 : 0;
    P.fast = (S->opt.law == 0 && S->inv_lambda == (1ull << 32) && S->opt.tie_bits == 0 && S->fr.nb == 0 &&
              S->N < ((int64_t)1 << 32)) ? 1 : 0;
    {   // parity of the shard's first tile row in global tile coordinates (colouring only)
        const int t0 = sh.g.ndim == 2 ? sh.g.y0 / S->tile[1] : sh.g.z0 / S->tile[2];
        P.row_par0 = t0 & 1;
    }
    for (int i = 0; i < 14; ++i) P.thr[i] = S->thr[i];
    P.tile_hist = sh.tile_hist;
    P.tmap = sh.tmap;
    P.box_ok = sh.box_ok;
    for (int i = 0; i < 16; ++i) P.clsw[i] = i < 14 ? (unsigned int)(S->thr[i] >> 16) : 0u;
    P.cls_lim = S->cls_lim;
    return P;
}

// TMA tensor map of a shard's words with the tile box (tile + 2-word x halo + 1-cell y / z halo):
// interior tiles are staged by one cp.async.bulk.tensor (driver entry point, no libcuda link)
void encode_tile_box(aca_sim* S, Shard& sh) {
    static void* fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            fn = nullptr;
        }
    }
    sh.box_ok = 0;
    if (!fn || getenv("ACA_NO_TMA_BOX") || (sh.g.nx & 1)) return;
    const int nd = sh.g.ndim;
    cuuint64_t dims[3] = {(cuuint64_t)sh.g.nx, (cuuint64_t)sh.g.ny, (cuuint64_t)sh.g.nz};
    cuuint64_t strides[2] = {(cuuint64_t)sh.g.nx * 8, (cuuint64_t)sh.g.nx * sh.g.ny * 8};
    cuuint32_t box[3] = {(cuuint32_t)S->tile[0] + 4, (cuuint32_t)S->tile[1] + 2, (cuuint32_t)S->tile[2] + 2};
    cuuint32_t estr[3] = {1, 1, 1};
    if (box[0] > 256 || box[1] > 256 || box[2] > 256) return;
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    // L2 fetch granule of the box loads: 64 B. The box's rows start 16 B before a tile row (the
    // 2-word x halo), so a 256 B granule fetched 2 x 240 B of the neighbours per row that no tile
    // of the launch uses (c3: 1.88 -> 1.37 GB of DRAM reads per launch, +1.4 %; r02g promo A/B)
    CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    if (const char* e = getenv("ACA_TMA_PROMO")) {   // ablation: 0 (none), 64, 128, 256
        const int v = atoi(e);
        promo = v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
              : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    }
    CUresult r = enc(&sh.tmap, CU_TENSOR_MAP_DATA_TYPE_UINT64, (cuuint32_t)nd, sh.words, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    sh.box_ok = r == CUDA_SUCCESS ? 1 : 0;
}

// a10 class bookkeeping: recount every tile's class histogram from the current state
int class_refresh(aca_sim* S) {
    if (!S->cls) return ACA_OK;
    for (auto& sh : S->shards) {
        const KParams P = make_params(S, sh);
        const int nt = sh.tiles_x * sh.tiles_y * sh.tiles_z;
        class_refresh_kernel<256><<<nt, 256, 0, S->stream>>>(P, S->tile[0], S->tile[1], S->tile[2]);
        CK(cudaGetLastError());
    }
    S->cls_stale = false;
    return ACA_OK;
}

// exchange of the sharded-axis boundary rows/planes (virtual shards: D2D copies;
// multi-process: NCCL send/recv to ring neighbours)
int exchange(aca_sim* S) {
    if (S->use_nccl) {
        NcclApi& api = nccl();
        Shard& sh = S->shards[0];
        const int up = (S->rank + 1) % S->world, dn = (S->rank + S->world - 1) % S->world;
        const size_t bytes = sh.face * 8;
        const unsigned long long* first = sh.words;
        const unsigned long long* last = sh.words + (sh.n - sh.face);
        api.gstart();
        api.send(first, bytes, NCCL_UINT8, dn, S->comm, S->stream);   // my first row -> below's halo_hi
        api.send(last, bytes, NCCL_UINT8, up, S->comm, S->stream);    // my last row -> above's halo_lo
        api.recv(sh.halo_hi, bytes, NCCL_UINT8, up, S->comm, S->stream);
        api.recv(sh.halo_lo, bytes, NCCL_UINT8, dn, S->comm, S->stream);
        int r = api.gend();
        if (r != 0) return fail(ACA_ENCCL, "NCCL halo exchange failed: %d", r);
        return ACA_OK;
    }
    if (S->G == 1) return ACA_OK;
    for (int s = 0; s < S->G; ++s) {
        Shard& a = S->shards[s];
        Shard& up = S->shards[(s + 1) % S->G];
        Shard& dn = S->shards[(s + S->G - 1) % S->G];
        CK(cudaMemcpyAsync(dn.halo_hi, a.words, a.face * 8, cudaMemcpyDeviceToDevice, S->stream));
        CK(cudaMemcpyAsync(up.halo_lo, a.words + (a.n - a.face), a.face * 8, cudaMemcpyDeviceToDevice,
                           S->stream));
    }
    return ACA_OK;
}

// One outer round (sweep): every tile once. Checkerboard mode: two launches, colour 0 then
// colour 1, with a halo exchange before each.
int launch_round(aca_sim* S) {
    for (int ph = S->phased ? 0 : -1; ph < (S->phased ? 2 : 0); ++ph) {
        if (!S->push) {   // push mode: the kernels store boundary rows into the neighbours' halos
            int rc = exchange(S);
            if (rc) return rc;
        }
        for (auto& sh : S->shards) {
            KParams P = make_params(S, sh);
            P.phase = ph;
            void* args[] = {&P};
            const int ntiles = ph < 0 ? sh.tiles_x * sh.tiles_y * sh.tiles_z
                                      : ((sh.tiles_x + 1) / 2) * sh.tiles_y * sh.tiles_z;
            dim3 grid = S->whole ? dim3(1)
                                 : dim3(S->persistent_ctas > 0 ? std::min(ntiles, S->persistent_ctas) : ntiles);
            void* fn = (S->kern_gen && !P.fast) ? S->kern_gen : S->kern;
            CK(cudaLaunchKernel(fn, grid, dim3(S->nthreads), args, S->smem, S->stream));
            if (S->sync_debug) {   // ACA_SYNC_DEBUG=1: locate a failing launch (no graphs)
                cudaError_t e = cudaStreamSynchronize(S->stream);
                if (e != cudaSuccess && S->h_dbg && S->h_dbg[0])
                    return fail(ACA_ECUDA, "tile launch failed (phase %d, launch %llu): %s; first failed check line %llu a=%llu b=%llu thread %llu",
                                ph, (unsigned long long)S->kernel_launches, cudaGetErrorString(e), S->h_dbg[0],
                                S->h_dbg[1], S->h_dbg[2], S->h_dbg[3]);
                if (e != cudaSuccess) {
                    if (S->h_trace && P.dbg_trace) {
                        FILE* f = fopen("gpurun_out/trace.txt", "w");
                        for (int i = 0; i < 148 * 32 && f; ++i)
                            fprintf(f, "%d %d %llu %llu %llx\n", i / 32, i % 32, S->h_trace[2 * i], S->h_trace[2 * i + 1] >> 56,
                                    S->h_trace[2 * i + 1] & 0xffffffffffffffull);
                        if (f) fclose(f);
                    }
                    return fail(ACA_ECUDA, "tile launch failed (phase %d, launch %llu): %s", ph,
                                (unsigned long long)S->kernel_launches, cudaGetErrorString(e));
                }
                Ctl c;
                CK(cudaMemcpy(&c, sh.ctl, sizeof c, cudaMemcpyDeviceToHost));
                if (c.dbg_line)
                    return fail(ACA_ESTATE, "device check failed at aca_tile.cuh:%u (a = %llu, b = %llu; phase %d, launch %llu)",
                                c.dbg_line, c.dbg_a, c.dbg_b, ph, (unsigned long long)S->kernel_launches);
            }
        }
        if (ph < 0) break;
    }
    return ACA_OK;
}

void drop_graph(aca_sim* S) {
    if (S->graph) cudaGraphExecDestroy(S->graph);
    S->graph = nullptr;
    S->graph_stale = false;
}

int build_graph(aca_sim* S) {
    if (S->graph && !S->graph_stale) return ACA_OK;
    if (S->use_nccl || S->sync_debug) return ACA_OK;   // NCCL path / ACA_SYNC_DEBUG: direct launches
    cudaGraph_t g = nullptr;
    if (cudaStreamBeginCapture(S->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        cudaGetLastError();
        drop_graph(S);
        return ACA_OK;
    }
    int rc = ACA_OK;
    for (int k = 0; k < S->K && rc == ACA_OK; ++k) rc = launch_round(S);
    cudaError_t e = cudaStreamEndCapture(S->stream, &g);
    if (rc != ACA_OK || e != cudaSuccess) {
        cudaGetLastError();
        if (g) cudaGraphDestroy(g);
        drop_graph(S);
        return ACA_OK;   // fall back to direct launches (same kernels)
    }
    if (S->graph) {   // stale parameters only: update the instantiated graph in place (no re-instantiation)
        cudaGraphExecUpdateResultInfo info;
        if (cudaGraphExecUpdate(S->graph, g, &info) == cudaSuccess) {
            cudaGraphDestroy(g);
            S->graph_stale = false;
            return ACA_OK;
        }
        cudaGetLastError();
        drop_graph(S);
    }
    e = cudaGraphInstantiate(&S->graph, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
        cudaGetLastError();
        S->graph = nullptr;
    }
    S->graph_rounds = S->K;
    return ACA_OK;
}

int sync_ctl(aca_sim* S) {
    for (size_t i = 0; i < S->shards.size(); ++i)
        CK(cudaMemcpyAsync(&S->h_ctl[i], S->shards[i].ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, S->stream));
    CK(cudaStreamSynchronize(S->stream));
    return ACA_OK;
}

int ensure_scratch(aca_sim* S, size_t bytes) {
    if (S->scratch_bytes >= bytes) return ACA_OK;
    if (S->scratch) cudaFree(S->scratch);
    S->scratch = nullptr;
    S->scratch_bytes = 0;
    CK(cudaMalloc(&S->scratch, bytes));
    S->scratch_bytes = bytes;
    return ACA_OK;
}

int check_count(const aca_sim* S, size_t count, const void* p) {
    if (!S) return fail(ACA_EINVAL, "null handle");
    if (!p) return fail(ACA_EINVAL, "null buffer");
    size_t n = 0;
    for (auto& sh : S->shards) n += sh.n;
    if (count != n) return fail(ACA_EINVAL, "count %zu != number of cells %zu", count, n);
    return ACA_OK;
}

constexpr size_t CHUNK = (size_t)1 << 25;   // cells per getter chunk (256 MB of u64)

int init_peer_halos(aca_sim* S);

// P5 initial state on the device + zeroed control blocks.
int init_state(aca_sim* S) {
    S->cls_stale = true;
    RoundKeys K;
    philox_round_keys((uint32_t)(S->seed & 0xffffffffu), (uint32_t)(S->seed >> 32), K.rk);
    for (auto& sh : S->shards) {
        CK(cudaMemsetAsync(sh.ctl, 0, sizeof(Ctl), S->stream));
        init_kernel<<<1184, 256, 0, S->stream>>>(sh.words, sh.g, S->d_lr, K, S->thr_init, S->inv_lambda,
                                                  S->opt.tie_bits, (unsigned long long)sh.n, S->opt.law);
        CK(cudaGetLastError());
    }
    S->T_last = 0;
    S->t_hi = S->max_delta + 1;
    if (S->ipc && S->shards[0].stats_lo) return init_peer_halos(S);
    return ACA_OK;
}

// Multi-process (IPC) handles after a (re)initialisation: the neighbours' boundary rows are
// their P5 initial states, a function of (seed, cell) alone, so each rank fills its halo buffers
// (and the statistics' snapshot of them) itself: the P5 kernel on a one-row (one-plane) shard
// at the neighbour's global offset.
int init_peer_halos(aca_sim* S) {
    RoundKeys K;
    philox_round_keys((uint32_t)(S->seed & 0xffffffffu), (uint32_t)(S->seed >> 32), K.rk);
    Shard& sh = S->shards[0];
    const bool d2 = sh.g.ndim == 2;
    const int n_axis = d2 ? sh.g.NY : sh.g.NZ, a0 = d2 ? sh.g.y0 : sh.g.z0, na = d2 ? sh.g.ny : sh.g.nz;
    for (int side = 0; side < 2; ++side) {
        Geo gh = sh.g;
        const int at = side == 0 ? (a0 - 1 + n_axis) % n_axis : (a0 + na) % n_axis;
        if (d2) { gh.ny = 1; gh.y0 = at; } else { gh.nz = 1; gh.z0 = at; }
        unsigned long long* dst = side == 0 ? sh.halo_lo : sh.halo_hi;
        init_kernel<<<148, 256, 0, S->stream>>>(dst, gh, S->d_lr, K, S->thr_init, S->inv_lambda, S->opt.tie_bits,
                                                 (unsigned long long)sh.face, S->opt.law);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(side == 0 ? sh.stats_lo : sh.stats_hi, dst, sh.face * 8, cudaMemcpyDeviceToDevice, S->stream));
    }
    S->snap_valid = true;
    return ACA_OK;
}

// Device reductions over all shards (the halos are refreshed first for the bond sum).
int device_stats(aca_sim* S) {
    StatAcc init{0, 0, 0, ~0ull, 0, 0};
    *S->h_stat = init;
    CK(cudaMemcpyAsync(S->d_stat, S->h_stat, sizeof(StatAcc), cudaMemcpyHostToDevice, S->stream));
    int rc = exchange(S);
    if (rc) return rc;
    if (S->ipc && !S->snap_valid)
        return fail(ACA_ESTATE, "multi-process statistics after set_state / set_spins need a run_until first "
                                "(the neighbours' boundary rows are not known yet)");
    for (auto& sh : S->shards) {
        KParams P = make_params(S, sh);
        if (S->ipc) {   // the neighbours' rows as of the end of the last run (or their P5 state)
            P.halo_lo = sh.stats_lo;
            P.halo_hi = sh.stats_hi;
        }
        stats_kernel<256><<<1184, 256, 0, S->stream>>>(P, S->d_stat, (unsigned long long)sh.n);
        CK(cudaGetLastError());
    }
    CK(cudaMemcpyAsync(S->h_stat, S->d_stat, sizeof(StatAcc), cudaMemcpyDeviceToHost, S->stream));
    CK(cudaStreamSynchronize(S->stream));
    return ACA_OK;
}

// Choose the (t, n) split of the packed word for horizon Tq: the fewest time bits that hold both
// every time the run can produce (< Tq + max_delta) and every time already stored (< t_hi),
// every remaining bit for the counter (capped at 31); repack if it changed. Growing the counter
// field shrinks the time field, which is safe because tb covers t_hi; shrinking it is checked
// against the largest stored counter.
int fit_layout(aca_sim* S, uint64_t Tq) {
    const unsigned long long tmax = (unsigned long long)Tq + S->max_delta;
    if (tmax < (unsigned long long)Tq) return fail(ACA_ERANGE, "time horizon overflows 64 bits");
    const int tb = bits_for(std::max<unsigned long long>(tmax, S->t_hi));
    int nb = 63 - tb;
    if (nb > 31) nb = 31;
    // tests only: a narrower counter field widens the time quantum of the words' high halves, so
    // small lattices see the high-half ties (and their exact passes) that full-size runs see
    if (const char* e = getenv("ACA_NB_CAP")) nb = std::min(nb, std::max(1, atoi(e)));
    if (nb < 1) return fail(ACA_ERANGE, "time bits (%d) leave no room for the counter", tb);
    if (nb == S->NB) return ACA_OK;
    if (nb < S->NB) {   // shrinking the counter field: every current counter must fit
        int rc = device_stats(S);
        if (rc) return rc;
        if (S->h_stat->nmax >= (1ull << nb) - 1ull)
            return fail(ACA_ERANGE, "event counters (max %llu) do not fit the %d bits left by T", S->h_stat->nmax, nb);
    }
    const int old_nb = S->NB;
    S->NB = nb;
    S->TB = 63 - nb;
    set_geo_layout(S);
    for (auto& sh : S->shards) {
        Geo ga = sh.g;
        ga.NB = old_nb;
        ga.TSH = old_nb + 1;
        ga.nbmask = (1u << old_nb) - 1u;
        repack_kernel<<<1184, 256, 0, S->stream>>>(sh.words, ga, sh.g, (unsigned long long)sh.n);
        CK(cudaGetLastError());
    }
    drop_graph(S);   // kernel parameters (layout) changed
    return ACA_OK;
}

}  // namespace

// ============================================================================ C ABI
extern "C" {

const char* aca_last_error(void) { return g_err.c_str(); }

int aca_default_options(aca_options* o) {
    if (!o) return fail(ACA_EINVAL, "null options");
    memset(o, 0, sizeof *o);
    o->struct_size = sizeof(aca_options);
    o->init_q = 0.5;
    o->device = -1;
    o->shards = 1;
    o->rank = 0;
    o->world = 1;
    o->event_hash = 1;
    return ACA_OK;
}

int64_t aca_num_cells(const aca_sim* S) {
    if (!S) return -1;
    int64_t n = 0;
    for (auto& sh : S->shards) n += (int64_t)sh.n;
    return n;
}

void aca_destroy(aca_sim* S) {
    if (!S) return;
    if (S->stream) cudaStreamSynchronize(S->stream);
    drop_graph(S);
    for (auto& sh : S->shards) {
        cudaFree(sh.words);
        cudaFree(sh.halo_lo);
        cudaFree(sh.halo_hi);
        cudaFree(sh.ctl);
        cudaFree(sh.stats_lo);
        cudaFree(sh.stats_hi);
        cudaFree(sh.tile_hist);
    }
    if (S->comm && nccl().ok) nccl().destroy(S->comm);
    for (void* p : S->ipc_opened) cudaIpcCloseMemHandle(p);
    cudaFree(S->d_slot);
    cudaFree(S->d_lr);
    cudaFree(S->scratch);
    cudaFree(S->d_stat);
    cudaFree(S->frame_ring);
    if (S->h_ctl) cudaFreeHost(S->h_ctl);
    if (S->h_stat) cudaFreeHost(S->h_stat);
    if (S->ev0) cudaEventDestroy(S->ev0);
    if (S->ev1) cudaEventDestroy(S->ev1);
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b)
            if (S->evb[a][b]) cudaEventDestroy(S->evb[a][b]);
    cudaFree(S->d_flag);
    if (S->h_flag) cudaFreeHost(S->h_flag);
    if (S->cstream) cudaStreamSynchronize(S->cstream);
    for (int a = 0; a < 2; ++a) {
        cudaFree(S->stage_in[a]);
        cudaFree(S->stage_out[a]);
        for (cudaEvent_t e : {S->ev_h2d[a], S->ev_pack[a], S->ev_unp[a], S->ev_d2h[a]})
            if (e) cudaEventDestroy(e);
    }
    if (S->cstream) cudaStreamDestroy(S->cstream);
    if (S->own_stream && S->stream) cudaStreamDestroy(S->stream);
    delete S;
}

int aca_create(aca_sim** out, int ndim, const int64_t* dims, int periodic, double lambda, double beta,
               double J, double h, int rule, uint64_t seed, const aca_options* opt_in) {
    if (!out) return fail(ACA_EINVAL, "null out");
    *out = nullptr;
    if (ndim != 2 && ndim != 3) return fail(ACA_EINVAL, "ndim must be 2 or 3 (got %d)", ndim);
    if (!dims) return fail(ACA_EINVAL, "null dims");
    if (periodic != 1) return fail(ACA_EINVAL, "only periodic boundaries are supported (periodic=1)");
    if (!(lambda > 0) || !std::isfinite(lambda)) return fail(ACA_EINVAL, "lambda must be > 0 and finite");
    if (!(lambda >= 1.0 / 4294967296.0 * 2) || lambda > 4294967296.0)
        return fail(ACA_EINVAL, "lambda outside [2^-31, 2^32]");
    if (!(beta >= 0) || !std::isfinite(beta)) return fail(ACA_EINVAL, "beta must be >= 0 and finite");
    if (!std::isfinite(J) || !std::isfinite(h)) return fail(ACA_EINVAL, "J and h must be finite");
    if (rule != ACA_HEATBATH && rule != ACA_METROPOLIS && !(rule == ACA_LIFE && ndim == 2))
        return fail(ACA_EINVAL, "rule must be 0 (heat-bath), 1 (Metropolis) or 2 (Game of Life, 2-D)");
    aca_options opt;
    aca_default_options(&opt);
    if (opt_in) {
        if (opt_in->struct_size != sizeof(aca_options))
            return fail(ACA_EINVAL, "aca_options.struct_size %u != %zu", opt_in->struct_size, sizeof(aca_options));
        opt = *opt_in;
    }
    if (!(opt.init_q >= 0 && opt.init_q <= 1)) return fail(ACA_EINVAL, "init_q must be in [0, 1]");
    if (opt.tie_bits < 0 || opt.tie_bits > 40) return fail(ACA_EINVAL, "tie_bits must be in [0, 40]");
    if (opt.law < 0 || opt.law > 4)
        return fail(ACA_EINVAL, "law must be 0 (Poisson), 1 (uniform), 2 (r^1/8), 3 (Gaussian period) or 4 (fixed "
                                "Gaussian period per cell)");
    if (rule == ACA_LIFE && (opt.early_reject || opt.sync_rounds))
        return fail(ACA_EINVAL, "the Game of Life rule has no early rejection / sync-round kernel");
    if (opt.shards < 1) opt.shards = 1;
    if (opt.world < 1 || opt.rank < 0 || opt.rank >= opt.world) return fail(ACA_EINVAL, "bad rank/world");
    if ((opt.world > 1 || opt.nccl_id) && opt.shards != 1)
        return fail(ACA_EINVAL, "NCCL (multi-process) handles use shards = 1");
    if (opt.world > 1 && !opt.nccl_id && opt.halo_mode != 0)
        return fail(ACA_EINVAL, "world > 1 with halo_mode 1 (exchange) needs nccl_id");
    if (opt.rounds_per_launch < 0 || opt.launches_per_check < 0) return fail(ACA_EINVAL, "negative counts");
    if (opt.variant != 0)
        return fail(ACA_EINVAL, "variant must be 0 (the kernel ablations of round 1 were retired; DESIGN.md section 6)");
    if (opt.max_ctas < 0) return fail(ACA_EINVAL, "max_ctas must be >= 0");
    if (!(opt.lag >= 0) || !std::isfinite(opt.lag)) return fail(ACA_EINVAL, "lag must be >= 0 and finite (0 = off)");
    if (opt.class_book != 0 && opt.class_book != 1) return fail(ACA_EINVAL, "class_book must be 0 or 1");
    if (opt.class_book && (rule == ACA_LIFE || opt.sync_rounds || opt.whole_lattice == 1))
        return fail(ACA_EINVAL, "class_book needs the persistent tile kernel of an Ising rule");
    if (!std::isfinite(opt.class_wmax)) return fail(ACA_EINVAL, "class_wmax must be finite");

    int64_t N = 1;
    for (int a = 0; a < ndim; ++a) {
        if (dims[a] < 2) return fail(ACA_EINVAL, "every dimension must be >= 2 (dims[%d]=%lld)", a, (long long)dims[a]);
        if (dims[a] > (1 << 30)) return fail(ACA_EINVAL, "dimension too large");
        N *= dims[a];
        if (N > (int64_t)1 << 40) return fail(ACA_EINVAL, "lattice too large");
    }
    const int saxis = ndim - 1;                       // sharded axis
    const int parts = opt.world > 1 ? opt.world : opt.shards;
    if (dims[saxis] % parts != 0 || dims[saxis] / parts < 1)
        return fail(ACA_EINVAL, "%d shards do not divide the sharded axis (%lld)", parts, (long long)dims[saxis]);

    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(ACA_ENODEV, "no CUDA device (the library has no CPU fallback)");
    }

    aca_sim* S = new aca_sim();
    S->ndim = ndim;
    for (int a = 0; a < ndim; ++a) S->dims[a] = dims[a];
    S->N = N;
    S->lambda = lambda; S->beta = beta; S->J = J; S->h = h; S->rule = rule; S->seed = seed;
    S->opt = opt;
    S->device = opt.device >= 0 ? opt.device : -1;
    if (S->device < 0) {
        if (cudaGetDevice(&S->device) != cudaSuccess) { delete S; return fail(ACA_ECUDA, "cudaGetDevice"); }
    }
    if (cudaSetDevice(S->device) != cudaSuccess) { delete S; return fail(ACA_ECUDA, "cudaSetDevice(%d)", S->device); }
    S->rank = opt.world > 1 ? opt.rank : 0;
    S->world = opt.world;
    // world > 1, halo_mode 0: push over CUDA IPC mappings of the neighbours' halos (no NCCL);
    // otherwise an nccl_id selects NCCL send/recv exchange (world 1 + nccl_id: the ring of one)
    S->ipc = opt.world > 1 && opt.halo_mode == 0;
    S->use_nccl = !S->ipc && opt.nccl_id != nullptr;
    S->G = opt.world > 1 ? 1 : opt.shards;
    S->sync = opt.sync_rounds != 0;
    S->rounds = opt.rounds_per_launch > 0 ? opt.rounds_per_launch : 5;   // measured best (c3, c4, c5) with checkerboard sweeps
    S->K = opt.launches_per_check > 0 ? opt.launches_per_check : 16;
    if (const char* e = getenv("ACA_SYNC_DEBUG")) S->sync_debug = atoi(e) != 0;
    if (S->sync_debug && cudaHostAlloc((void**)&S->h_dbg, 64, cudaHostAllocMapped) == cudaSuccess) memset(S->h_dbg, 0, 64);
    if (const char* e = getenv("ACA_TRACE_FROM")) {
        S->trace_from = atoll(e);
        if (cudaHostAlloc((void**)&S->h_trace, 148 * 32 * 16, cudaHostAllocMapped) != cudaSuccess) S->h_trace = nullptr;
        else memset(S->h_trace, 0, 148 * 32 * 16);
    }

    // P3 constants, P4 table, P5 threshold, packed-word layout
    S->inv_lambda = (unsigned long long)std::floor(4294967296.0 / lambda + 0.5);
    if (opt.lag > 0) S->lag_q = std::max(1ull, (unsigned long long)std::floor(opt.lag / lambda * 4294967296.0 + 0.5));
    flip_table(ndim, beta, J, h, rule, S->thr);
    early_table(ndim, S->thr, opt.early_reject != 0, S->thm);
    S->bulk = 1;   // one committed arrival per cell per fire step: longer in-thread chains
                   // diverge within the warp (measured: bulk 4/32 are 1.8-2x slower on c5)
    if (const char* e = getenv("ACA_BULK")) S->bulk = std::max(1, atoi(e));
    S->thr_init = (unsigned long long)std::floor(opt.init_q * 4294967296.0);
    {
        // largest unscaled increment of the law: NLOG-2(1) for Poisson, < 2^32 otherwise
        // (laws 3 and 4: 1 + 6.34/4 < 3 periods)
        const unsigned long long umax = opt.law == 0 ? 190530846196ull : opt.law >= 3 ? (3ull << 32) : (1ull << 32);
        const unsigned __int128 p = (unsigned __int128)umax * S->inv_lambda;
        S->max_delta = (unsigned long long)(p >> 32) + 1 + (opt.tie_bits ? (1ull << opt.tie_bits) : 0ull);
        const int tb = bits_for(S->max_delta);
        int nb = 63 - tb;
        if (nb > 31) nb = 31;
        if (nb < 1) { delete S; return fail(ACA_ERANGE, "lambda leaves no room in the packed word"); }
        S->NB = nb;
        S->TB = 63 - nb;
        S->t_hi = S->max_delta + 1;
    }

    auto bail = [&](int code) { aca_destroy(S); return code; };
    if (opt.stream) {
        S->stream = (cudaStream_t)opt.stream;
    } else {
        if (cudaStreamCreateWithFlags(&S->stream, cudaStreamNonBlocking) != cudaSuccess)
            return bail(fail(ACA_ECUDA, "cudaStreamCreate"));
        S->own_stream = true;
    }
    if (cudaMalloc(&S->d_lr, sizeof(ACA_NLOG_LR)) != cudaSuccess) return bail(fail(ACA_ENOMEM, "cudaMalloc lr"));
    if (cudaMemcpy(S->d_lr, ACA_NLOG_LR, sizeof(ACA_NLOG_LR), cudaMemcpyHostToDevice) != cudaSuccess)
        return bail(fail(ACA_ECUDA, "copy nlog table"));
    if (cudaMalloc(&S->d_stat, sizeof(StatAcc)) != cudaSuccess) return bail(fail(ACA_ENOMEM, "cudaMalloc stat"));
    if (cudaMallocHost(&S->h_stat, sizeof(StatAcc)) != cudaSuccess) return bail(fail(ACA_ENOMEM, "pinned stat"));
    if (cudaEventCreate(&S->ev0) != cudaSuccess || cudaEventCreate(&S->ev1) != cudaSuccess)
        return bail(fail(ACA_ECUDA, "cudaEventCreate"));
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b)
            if (cudaEventCreate(&S->evb[a][b]) != cudaSuccess) return bail(fail(ACA_ECUDA, "cudaEventCreate"));
    if (cudaMalloc(&S->d_flag, 8) != cudaSuccess || cudaMallocHost(&S->h_flag, 8) != cudaSuccess)
        return bail(fail(ACA_ENOMEM, "flag"));

    // kernel selection
    int dev_smem = 0;
    cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, S->device);
    const bool single = (S->G == 1 && S->world == 1 && !S->use_nccl);
    S->whole = false;
    if (single && opt.whole_lattice >= 0 && !opt.class_book) {
        const bool fits = whole_smem(N, S->sync) <= (size_t)dev_smem;
        if (opt.whole_lattice == 1 && !fits) return bail(fail(ACA_EINVAL, "lattice too large for whole_lattice"));
        S->whole = fits && (opt.whole_lattice == 1 || N <= 8192);
    }
    if (S->whole) {
        S->kern = S->sync ? (void*)whole_kernel<WHOLE_NT, true> : (void*)whole_kernel<WHOLE_NT, false>;
        S->nthreads = WHOLE_NT;
        S->smem = whole_smem(N, S->sync);
        S->rounds = 1 << 30;
    } else {
        int tx = opt.tile[0], ty = opt.tile[1], tz = opt.tile[2];
        if (tx == 0 && ty == 0 && tz == 0) {
            if (ndim == 2) { tx = 64; ty = 64; tz = 1; }
            else { tx = 32; ty = 16; tz = 8; }
        }
        if (ndim == 2) tz = 1;
        const TileKey* sel = nullptr;
        int want_ntg = 0;
        if (const char* nt_env = getenv("ACA_TILE_NT")) want_ntg = atoi(nt_env);   // ablation: group size of a shape
        if (want_ntg == 0 && ndim == 2 && tx == 64 && ty == 64) {
            // few tiles per launch (config 2: 128 per colour on 148 SMs): 512 threads per 64x64
            // tile halve each round's latency; with many tiles 256-thread groups are faster
            int nsm = 148;
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, S->device);
            const int64_t rows = dims[1] / parts;
            const int64_t tiles = ((dims[0] + 63) / 64) * ((rows + 63) / 64);
            if ((int64_t)dims[0] * rows >= ((int64_t)1 << 20) && tiles / 2 < 2 * (int64_t)nsm) want_ntg = 512;
        }
        for (const auto& k : kTiles)
            if (k.ndim == ndim && k.tx == tx && k.ty == ty && k.tz == tz && (want_ntg == 0 || k.ntg == want_ntg) && !sel)
                sel = &k;
        if (!sel) return bail(fail(ACA_EINVAL, "unsupported tile %dx%dx%d for ndim %d", tx, ty, tz, ndim));
        S->tile[0] = tx; S->tile[1] = ty; S->tile[2] = tz;
        if (S->sync) {   // fig:s1c1pe reference: one CTA per tile, all tiles in one launch
            S->kern = sel->fn_sync;
            S->nthreads = sel->nt_sync;
            S->smem = sel->smem_sync;
        } else {
            const bool early = opt.early_reject != 0 && rule != ACA_LIFE;
            S->kern = rule == ACA_LIFE ? sel->fn_life : early ? sel->fn_early : sel->fn;
            S->kern_gen = rule == ACA_LIFE ? nullptr : early ? sel->fn_early_gen : sel->fn_gen;
            S->nthreads = early ? sel->nt_early : sel->nt;
            S->smem = early ? sel->smem_early : sel->smem;
            if (opt.class_book) {   // a10 per-tile class bookkeeping: the a10 or the plain path per tile visit
                if (!sel->fn_cls)
                    return bail(fail(ACA_EINVAL, "class_book needs the default tile (64x64 in 2-D, 32x16x8 in 3-D)"));
                S->cls = true;
                S->kern = sel->fn_cls;
                S->kern_gen = sel->fn_cls_gen;
                S->nthreads = sel->nt_early;
                S->smem = sel->smem_cls;
                // early path iff the tile's mean flip probability per arrival, sum_k |Gamma_k| p_k / cells,
                // is at most class_wmax (early_reject = 0: never; the histograms are still kept)
                const double cells = (double)tx * ty * tz, lim = std::floor(opt.class_wmax * 65536.0 * cells);
                S->cls_lim = (!early || opt.class_wmax < 0) ? -1 : (long long)std::min(lim, 4.0e18);
            }
            if (cudaFuncSetAttribute(S->kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S->smem) != cudaSuccess)
                return bail(fail(ACA_ECUDA, "smem attribute (tile)"));
            if (S->kern_gen &&
                cudaFuncSetAttribute(S->kern_gen, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S->smem) != cudaSuccess)
                return bail(fail(ACA_ECUDA, "smem attribute (tile, general arrival)"));
            int nsm = 0, occ = 0;
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, S->device);
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, S->kern, S->nthreads, S->smem) != cudaSuccess || occ < 1)
                return bail(fail(ACA_ECUDA, "occupancy query failed (%zu B shared memory, %d threads)", S->smem,
                                 S->nthreads));
            // persistent: one CTA per SM (as many as fit), optionally capped (max_ctas drives the
            // multi-tile-per-CTA buffer ring on small lattices)
            S->persistent_ctas = nsm * occ;
            if (opt.max_ctas > 0) S->persistent_ctas = std::min(S->persistent_ctas, opt.max_ctas);
            S->phased = opt.checkerboard >= 0;
        }
    }
    if (cudaFuncSetAttribute(S->kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S->smem) != cudaSuccess)
        return bail(fail(ACA_ECUDA, "smem attribute"));

    // shards
    const int64_t local = dims[saxis] / parts;
    S->shards.resize(S->G);
    for (int s = 0; s < S->G; ++s) {
        Shard& sh = S->shards[s];
        const int part = S->world > 1 ? S->rank : s;
        Geo& g = sh.g;
        g.ndim = ndim;
        g.nx = (int)dims[0];
        g.NY = (int)dims[1];
        g.NZ = ndim == 3 ? (int)dims[2] : 1;
        g.ny = ndim == 2 ? (int)local : (int)dims[1];
        g.nz = ndim == 3 ? (int)local : 1;
        g.y0 = ndim == 2 ? (int)(part * local) : 0;
        g.z0 = ndim == 3 ? (int)(part * local) : 0;
        g.sharded = parts > 1 || S->use_nccl;
        sh.n = (size_t)g.nx * g.ny * g.nz;
        sh.face = ndim == 2 ? (size_t)g.nx : (size_t)g.nx * g.ny;
        sh.tiles_x = (g.nx + S->tile[0] - 1) / S->tile[0];
        sh.tiles_y = (g.ny + S->tile[1] - 1) / S->tile[1];
        sh.tiles_z = ndim == 3 ? (g.nz + S->tile[2] - 1) / S->tile[2] : 1;
        if (cudaMalloc(&sh.words, sh.n * 8) != cudaSuccess || cudaMalloc(&sh.ctl, sizeof(Ctl)) != cudaSuccess)
            return bail(fail(ACA_ENOMEM, "device allocation of %zu cells failed", sh.n));
        if (!S->whole && !S->sync) encode_tile_box(S, sh);
        if (S->cls &&
            cudaMalloc(&sh.tile_hist, (size_t)sh.tiles_x * sh.tiles_y * sh.tiles_z * 16 * sizeof(unsigned int)) != cudaSuccess)
            return bail(fail(ACA_ENOMEM, "tile class histograms"));
        if (g.sharded) {
            if (cudaMalloc(&sh.halo_lo, sh.face * 8) != cudaSuccess || cudaMalloc(&sh.halo_hi, sh.face * 8) != cudaSuccess)
                return bail(fail(ACA_ENOMEM, "halo allocation failed"));
        }
    }
    set_geo_layout(S);
    // push mode for virtual shards on this device (the persistent tile kernels store their
    // boundary rows into the neighbour shard's halo; multi-process handles use halo exchange)
    if (S->G > 1 && !S->use_nccl && S->persistent_ctas > 0 && opt.halo_mode == 0) {
        S->push = true;
        for (int s2 = 0; s2 < S->G; ++s2) {
            S->shards[s2].push_lo = S->shards[(s2 + S->G - 1) % S->G].halo_hi;
            S->shards[s2].push_hi = S->shards[(s2 + 1) % S->G].halo_lo;
        }
    }
    // resident-tile kernel: 2-D, one shard, whole 64 x 64 tiles, at most two tiles per colour per SM,
    // the plain test (no a10, no class bookkeeping, Ising rules), Poisson law at lambda = 1, no tie
    // stress, checkerboard sweeps (ACA_NO_RES=1: never, for ablations and parity tests)
    if (ndim == 2 && S->G == 1 && S->world == 1 && !S->use_nccl && !S->whole && !S->sync && !S->cls &&
        S->persistent_ctas > 0 && S->phased && S->tile[0] == 64 && S->tile[1] == 64 && dims[0] % 64 == 0 &&
        dims[1] % 64 == 0 && !opt.early_reject && rule != ACA_LIFE && opt.law == 0 && opt.tie_bits == 0 &&
        S->inv_lambda == (1ull << 32) && N < ((int64_t)1 << 32) && opt.max_ctas == 0 && !getenv("ACA_NO_RES")) {
        int nsm = 0, occ = 0;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, S->device);
        int nt = 512;
        if (const char* e = getenv("ACA_RES_NT")) nt = atoi(e) == 1024 ? 1024 : 512;   // ablation
        void* fn = nt == 1024 ? (void*)res_kernel<1024> : (void*)res_kernel<512>;
        const size_t sm = res_smem_bytes(nt);
        const int items = (int)((S->shards[0].tiles_x + 1) / 2) * S->shards[0].tiles_y;
        const int per = (items + nsm - 1) / nsm;
        if (per <= res_tiles_max() / 2 &&
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) == cudaSuccess &&
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, nt, sm) == cudaSuccess && occ >= 1) {
            S->res_nt = nt;
            S->res_fn = fn;
            S->res_ok = true;
            S->res_grid = (items + per - 1) / per;
            S->res_smem = sm;
        }
        cudaGetLastError();
    }
    if (int r = init_state(S)) return bail(r);
    if (cudaMallocHost(&S->h_ctl, 2 * sizeof(Ctl) * S->shards.size()) != cudaSuccess)
        return bail(fail(ACA_ENOMEM, "pinned ctl"));

    if (S->ipc && !(S->persistent_ctas > 0 && !S->whole))
        return bail(fail(ACA_EINVAL, "multi-process push mode needs the persistent tile kernel (not sync_rounds)"));
    if (S->ipc) {   // this rank's {epoch, active} slot, read by every rank through CUDA IPC
        if (cudaMalloc(&S->d_slot, 32) != cudaSuccess) return bail(fail(ACA_ENOMEM, "ipc slot"));
        if (cudaMemset(S->d_slot, 0, 32) != cudaSuccess) return bail(fail(ACA_ECUDA, "ipc slot"));
        Shard& sh0 = S->shards[0];
        if (cudaMalloc(&sh0.stats_lo, sh0.face * 8) != cudaSuccess || cudaMalloc(&sh0.stats_hi, sh0.face * 8) != cudaSuccess)
            return bail(fail(ACA_ENOMEM, "stats halo allocation failed"));
        if (int r = init_peer_halos(S)) return bail(r);
        S->push = true;   // push pointers are set by aca_ipc_import
    }
    if (S->use_nccl) {
        NcclApi& api = nccl();
        if (!api.ok) return bail(fail(ACA_ENCCL, "NCCL symbols not found in the process (load torch.distributed nccl first)"));
        ncclUniqueId_t id;
        memcpy(&id, opt.nccl_id, sizeof id);
        int r = api.init(&S->comm, S->world, id, S->rank);
        if (r != 0) return bail(fail(ACA_ENCCL, "ncclCommInitRank failed: %d", r));
    }
    if (cudaStreamSynchronize(S->stream) != cudaSuccess)
        return bail(fail(ACA_ECUDA, "init sync: %s", cudaGetErrorString(cudaGetLastError())));
    *out = S;
    return ACA_OK;
}

int aca_run_until_q32(aca_sim* S, uint64_t Tq) {
    if (!S) return fail(ACA_EINVAL, "null handle");
    if (Tq < S->T_last) return fail(ACA_ESTATE, "T decreased (%llu < %llu)", (unsigned long long)Tq, (unsigned long long)S->T_last);
    CK(cudaSetDevice(S->device));
    int rc = fit_layout(S, Tq);
    if (rc) return rc;
    S->T_last = Tq;
    S->t_hi = std::max<uint64_t>(S->t_hi, Tq + S->max_delta);   // every time the run can store
    const int TSH = S->NB + 1;
    // bounded lag: the first launch fires below min(T, global minimum time + lag); the tile
    // kernels then move the bound with the minimum (finish_launch). The minimum over all shards.
    unsigned long long wfirst = (unsigned long long)Tq << TSH, wmin0 = ~0ull;
    if (S->lag_q && !S->whole && !S->sync) {
        if (S->ipc) return fail(ACA_EINVAL, "the lag window is a single-process option");
        rc = device_stats(S);
        if (rc) return rc;
        const unsigned long long tmin = S->h_stat->tmin;
        if (tmin != ~0ull) {
            wmin0 = tmin << TSH;
            if (tmin + S->lag_q < Tq) wfirst = (tmin + S->lag_q) << TSH;
        }
    }
    for (size_t i = 0; i < S->shards.size(); ++i) {
        Ctl& h = S->h_ctl[i];
        h.wlim = wfirst;
        h.wlim_T = (unsigned long long)Tq << TSH;
        h.wmin[0] = h.wmin[1] = wmin0;
        CK(cudaMemcpyAsync(&S->shards[i].ctl->wlim, &h.wlim, sizeof(unsigned long long), cudaMemcpyHostToDevice,
                           S->stream));
        CK(cudaMemcpyAsync(&S->shards[i].ctl->wlim_T, &h.wlim_T, 3 * sizeof(unsigned long long), cudaMemcpyHostToDevice,
                           S->stream));
        CK(cudaMemsetAsync(&S->shards[i].ctl->done, 0, sizeof(unsigned int), S->stream));
    }
    if (S->ipc) {
        // multi-process push mode: write this rank's boundary rows into the neighbours' halos,
        // then wait until every rank has done so for this run (epoch barrier on the mapped
        // slots); from then on no rank waits for another until termination
        if (!S->ipc_ready) return fail(ACA_ESTATE, "multi-process push mode: call aca_ipc_import first");
        Shard& sh = S->shards[0];
        // every peer has snapshotted its halos at the end of the previous run before this rank's
        // boundary rows overwrite them
        for (int r = 0; r < S->world; ++r) {
            for (long spins = 0;; ++spins) {
                unsigned long long v[3];
                CK(cudaMemcpy(v, S->peer_slot[r], 24, cudaMemcpyDeviceToHost));
                if (v[2] >= S->epoch) break;
                if (spins > 20000000) return fail(ACA_ESTATE, "rank %d never finished run %llu", r, (unsigned long long)S->epoch);
                std::this_thread::sleep_for(std::chrono::microseconds(20));
            }
        }
        CK(cudaMemcpyAsync(sh.push_lo, sh.words, sh.face * 8, cudaMemcpyDeviceToDevice, S->stream));
        CK(cudaMemcpyAsync(sh.push_hi, sh.words + (sh.n - sh.face), sh.face * 8, cudaMemcpyDeviceToDevice, S->stream));
        CK(cudaStreamSynchronize(S->stream));
        S->epoch += 1;
        const unsigned long long mine[2] = {S->epoch, 1ull};
        CK(cudaMemcpy(S->d_slot, mine, 16, cudaMemcpyHostToDevice));
        for (int r = 0; r < S->world; ++r) {
            for (long spins = 0;; ++spins) {
                unsigned long long v[2];
                CK(cudaMemcpy(v, S->peer_slot[r], 16, cudaMemcpyDeviceToHost));
                if (v[0] >= S->epoch) break;
                if (spins > 20000000) return fail(ACA_ESTATE, "rank %d never reached run %llu", r, (unsigned long long)S->epoch);
                std::this_thread::sleep_for(std::chrono::microseconds(20));
            }
        }
    } else if (S->push) {   // push mode: fill the halos once; the kernels keep them current
        rc = exchange(S);
        if (rc) return rc;
    }
    if (S->cls && S->cls_stale) {   // the state was set from outside: recount the tiles' classes
        if (!S->push && !S->ipc) {
            rc = exchange(S);
            if (rc) return rc;
        }
        rc = class_refresh(S);
        if (rc) return rc;
    }
    // the resident-tile kernel when the run has the plain fast arrival and no lag window
    const bool use_res = S->res_ok && S->fr.nb == 0 && S->lag_q == 0;
    if (!use_res) {
        rc = build_graph(S);
        if (rc) return rc;
    }
    CK(cudaEventRecord(S->ev0, S->stream));
    const size_t nsh = S->shards.size();
    // One batch = K outer rounds (a CUDA-graph replay) followed by a copy of the control
    // blocks to pinned memory. Two batches are kept in flight so the GPU never idles while
    // the host inspects the previous batch; batches issued after termination are no-ops
    // (every launch returns at its first instruction when ctl->done is set).
    auto issue = [&](int slot) -> int {
        CK(cudaEventRecord(S->evb[slot][0], S->stream));
        if (use_res) {   // one launch runs to termination; a second one returns at once
            KParams P = make_params(S, S->shards[0]);
            P.phase = 0;
            void* args[] = {&P};
            CK(cudaLaunchCooperativeKernel(S->res_fn, dim3(S->res_grid), dim3(S->res_nt), args, S->res_smem,
                                           S->stream));
            S->kernel_launches += 1;
        } else if (S->graph) {
            CK(cudaGraphLaunch(S->graph, S->stream));
            S->kernel_launches += (uint64_t)S->graph_rounds * nsh * (S->phased ? 2 : 1);
        } else {
            for (int k = 0; k < S->K; ++k) {
                int r = launch_round(S);
                if (r) return r;
                S->kernel_launches += nsh * (S->phased ? 2 : 1);
            }
        }
        CK(cudaEventRecord(S->evb[slot][1], S->stream));
        for (size_t i = 0; i < nsh; ++i)
            CK(cudaMemcpyAsync(&S->h_ctl[slot * nsh + i], S->shards[i].ctl, sizeof(Ctl), cudaMemcpyDeviceToHost,
                               S->stream));
        CK(cudaEventRecord(S->evb[slot][2], S->stream));
        return ACA_OK;
    };
    auto retire = [&](int slot, bool* done) -> int {
        CK(cudaEventSynchronize(S->evb[slot][2]));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, S->evb[slot][0], S->evb[slot][1]));
        S->kernel_seconds += ms * 1e-3;
        bool d = true;
        for (size_t i = 0; i < nsh; ++i) d = d && S->h_ctl[slot * nsh + i].done;
        *done = d;
        return ACA_OK;
    };
    const bool pipelined = !S->use_nccl;
    rc = issue(0);
    if (rc) return rc;
    int outstanding = -1;      // pipelined: slot issued but not yet retired
    unsigned long long last_fired = ~0ull;
    int stall_batches = 0;
    for (int iter = 1;; ++iter) {
        const int cur = iter & 1, prev = cur ^ 1;
        if (pipelined) {
            rc = issue(cur);
            if (rc) return rc;
            outstanding = cur;
        }
        bool done = false;
        rc = retire(pipelined ? prev : 0, &done);
        if (rc) return rc;
        if (!done && S->world == 1) {
            // Every sweep fires at least the globally first pending arrival (fig:amcgen progress,
            // PAPER.md:820-823), so hundreds of batches without one fired arrival mean a broken
            // kernel, not a slow run: fail loudly instead of spinning. (A multi-process rank may
            // legitimately wait for its neighbours, so only single-process runs are checked.)
            unsigned long long f = 0;
            const int sl = pipelined ? prev : 0;
            for (size_t i = 0; i < nsh; ++i) f += S->h_ctl[sl * nsh + i].fired;
            stall_batches = f == last_fired ? stall_batches + 1 : 0;
            last_fired = f;
            if (stall_batches > 256)
                return fail(ACA_ESTATE, "no arrival fired in 256 batches of launches with cells still below T "
                                        "(a kernel fault: the method always makes progress)");
        }
        if (S->ipc && done) {
            // this rank has no cell below T any more (monotone: halos only grow); publish that
            // and wait, without issuing more batches, until every rank has. A rank whose epoch is
            // already ahead has seen all ranks done for this run.
            if (outstanding >= 0) {
                bool dummy;
                rc = retire(outstanding, &dummy);
                if (rc) return rc;
                outstanding = -1;
            }
            const unsigned long long act = 0ull;
            CK(cudaMemcpy(S->d_slot + 1, &act, 8, cudaMemcpyHostToDevice));
            for (long spins = 0;; ++spins) {
                bool all = true;
                for (int r = 0; r < S->world && all; ++r) {
                    unsigned long long v[2];
                    CK(cudaMemcpy(v, S->peer_slot[r], 16, cudaMemcpyDeviceToHost));
                    all = v[0] > S->epoch || (v[0] == S->epoch && v[1] == 0ull);
                }
                if (all) break;
                if (spins > 50000000) return fail(ACA_ESTATE, "peers never finished run %llu", (unsigned long long)S->epoch);
                std::this_thread::sleep_for(std::chrono::microseconds(20));
            }
        }
        if (S->use_nccl) {
            // every rank must agree: all-reduce of the local "still active" flag
            NcclApi& api = nccl();
            unsigned long long* d = S->d_flag;
            *S->h_flag = done ? 0ull : 1ull;
            CK(cudaMemcpyAsync(d, S->h_flag, 8, cudaMemcpyHostToDevice, S->stream));
            int r = api.allreduce(d, d, 1, NCCL_UINT64, NCCL_SUM, S->comm, S->stream);
            if (r != 0) return fail(ACA_ENCCL, "allreduce failed: %d", r);
            CK(cudaMemcpyAsync(S->h_flag, d, 8, cudaMemcpyDeviceToHost, S->stream));
            CK(cudaStreamSynchronize(S->stream));
            done = (*S->h_flag == 0);
            if (!done) {
                rc = issue(0);
                if (rc) return rc;
            }
        }
        if (done) break;
        if (iter > (1 << 26)) return fail(ACA_ESTATE, "no termination");
    }
    if (outstanding >= 0) {   // account the trailing (no-op) batch
        bool dummy;
        rc = retire(outstanding, &dummy);
        if (rc) return rc;
    }
    if (S->ipc) {
        // every rank is done, so every boundary row pushed into this rank's halos is final:
        // snapshot them for the statistics, then let the peers start their next run
        Shard& sh = S->shards[0];
        CK(cudaMemcpyAsync(sh.stats_lo, sh.halo_lo, sh.face * 8, cudaMemcpyDeviceToDevice, S->stream));
        CK(cudaMemcpyAsync(sh.stats_hi, sh.halo_hi, sh.face * 8, cudaMemcpyDeviceToDevice, S->stream));
        CK(cudaStreamSynchronize(S->stream));
        const unsigned long long snap = S->epoch;
        CK(cudaMemcpy(S->d_slot + 2, &snap, 8, cudaMemcpyHostToDevice));
        S->snap_valid = true;
    }
    CK(cudaEventRecord(S->ev1, S->stream));
    CK(cudaEventSynchronize(S->ev1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, S->ev0, S->ev1));
    S->gpu_seconds += ms * 1e-3;
    rc = sync_ctl(S);
    if (rc) return rc;
    for (size_t i = 0; i < nsh; ++i)
        if (S->h_ctl[i].overflow)
            return fail(ACA_ERANGE, "an event counter filled its %d-bit field; the run stopped early", S->NB);
    return ACA_OK;
}

int aca_nccl_unique_id(void* out128) {
    if (!out128) return fail(ACA_EINVAL, "null buffer");
    NcclApi& api = nccl();
    if (!api.ok || !api.uid) return fail(ACA_ENCCL, "NCCL not available in this process");
    ncclUniqueId_t id;
    int r = api.uid(&id);
    if (r != 0) return fail(ACA_ENCCL, "ncclGetUniqueId failed: %d", r);
    memcpy(out128, &id, sizeof id);
    return ACA_OK;
}

int aca_reset(aca_sim* S, uint64_t seed) {
    if (!S) return fail(ACA_EINVAL, "null handle");
    CK(cudaSetDevice(S->device));
    S->seed = seed;
    if (S->graph) S->graph_stale = true;   // the key is a kernel parameter: updated at the next run
    return init_state(S);
}

int aca_run_until(aca_sim* S, double T) {
    if (!S) return fail(ACA_EINVAL, "null handle");
    if (!(T >= 0) || !std::isfinite(T)) return fail(ACA_EINVAL, "T must be finite and >= 0");
    const double tq = std::floor(T * 4294967296.0 + 0.5);
    if (tq >= 18446744073709551616.0) return fail(ACA_ERANGE, "T too large");
    return aca_run_until_q32(S, (uint64_t)tq);
}

static int get_fields(aca_sim* S, int8_t* spins, uint64_t* times, uint32_t* counters, size_t count) {
    const void* any = spins ? (const void*)spins : times ? (const void*)times : (const void*)counters;
    int rc = check_count(S, count, any);
    if (rc) return rc;
    CK(cudaSetDevice(S->device));
    const size_t esz = times ? 8 : counters ? 4 : 1;
    rc = ensure_scratch(S, CHUNK * esz);
    if (rc) return rc;
    size_t off = 0;
    for (auto& sh : S->shards) {
        for (size_t b = 0; b < sh.n; b += CHUNK) {
            const size_t m = std::min(CHUNK, sh.n - b);
            unpack_kernel<<<592, 256, 0, S->stream>>>(sh.words + b, spins ? (int8_t*)S->scratch : nullptr,
                                                      times ? (unsigned long long*)S->scratch : nullptr,
                                                      counters ? (unsigned int*)S->scratch : nullptr, sh.g, m);
            CK(cudaGetLastError());
            void* dst = spins ? (void*)(spins + off + b) : times ? (void*)(times + off + b) : (void*)(counters + off + b);
            CK(cudaMemcpyAsync(dst, S->scratch, m * esz, cudaMemcpyDeviceToHost, S->stream));
            CK(cudaStreamSynchronize(S->stream));
        }
        off += sh.n;
    }
    return ACA_OK;
}

int aca_get_spins(aca_sim* S, int8_t* out, size_t count) { return get_fields(S, out, nullptr, nullptr, count); }
int aca_get_times(aca_sim* S, uint64_t* out, size_t count) { return get_fields(S, nullptr, out, nullptr, count); }
int aca_get_counters(aca_sim* S, uint32_t* out, size_t count) { return get_fields(S, nullptr, nullptr, out, count); }

int aca_get_cells(aca_sim* S, const int64_t* idx, size_t m, int8_t* spins, uint64_t* times, uint32_t* counters) {
    if (!S || (m && !idx)) return fail(ACA_EINVAL, "null argument");
    if (m == 0) return ACA_OK;
    const int64_t n = aca_num_cells(S);
    for (size_t i = 0; i < m; ++i)
        if (idx[i] < 0 || idx[i] >= n) return fail(ACA_EINVAL, "cell index %lld out of range", (long long)idx[i]);
    CK(cudaSetDevice(S->device));
    int rc = ensure_scratch(S, m * 16);
    if (rc) return rc;
    int64_t* didx = (int64_t*)S->scratch;
    unsigned long long* dw = (unsigned long long*)(didx + m);
    CK(cudaMemcpyAsync(didx, idx, m * 8, cudaMemcpyHostToDevice, S->stream));
    int64_t base = 0;
    for (auto& sh : S->shards) {
        gather_kernel<<<(unsigned)((m + 255) / 256), 256, 0, S->stream>>>(sh.words, didx, (unsigned long long)m, base,
                                                                         (long long)sh.n, dw);
        CK(cudaGetLastError());
        base += (int64_t)sh.n;
    }
    std::vector<unsigned long long> hw(m);
    CK(cudaMemcpyAsync(hw.data(), dw, m * 8, cudaMemcpyDeviceToHost, S->stream));
    CK(cudaStreamSynchronize(S->stream));
    const Geo& g = S->shards[0].g;
    for (size_t i = 0; i < m; ++i) {
        if (spins) spins[i] = (hw[i] & 1ull) ? 1 : -1;
        if (times) times[i] = w_time(hw[i], g);
        if (counters) counters[i] = w_count(hw[i], g);
    }
    return ACA_OK;
}

int aca_get_flip_table(const aca_sim* S, uint64_t* thr, size_t count) {
    if (!S || !thr) return fail(ACA_EINVAL, "null argument");
    const size_t n = 2 * (2 * S->ndim + 1);
    if (count != n) return fail(ACA_EINVAL, "flip table has %zu entries", n);
    for (size_t i = 0; i < n; ++i) thr[i] = S->thr[i];
    return ACA_OK;
}

int aca_get_stats(aca_sim* S, aca_stats* o) {
    if (!S || !o) return fail(ACA_EINVAL, "null argument");
    CK(cudaSetDevice(S->device));
    memset(o, 0, sizeof *o);
    int rc = device_stats(S);
    if (rc) return rc;
    rc = sync_ctl(S);
    if (rc) return rc;
    o->bond_sum = S->h_stat->bond;
    o->magnetisation = S->h_stat->mag;
    o->arrivals = S->h_stat->arrivals;
    o->t_min = S->h_stat->tmin;
    o->t_max = S->h_stat->tmax;
    for (size_t i = 0; i < S->shards.size(); ++i) {
        const Ctl& c = S->h_ctl[i];
        o->flips += c.flips;
        o->event_hash += c.hash;
        o->launches += c.launches;
        o->inner_rounds += c.inner_rounds;
        o->cells_tested += c.tested;
        o->cells_fired += c.fired;
        o->tile_visits_early += c.visits_early;
        o->tile_visits_plain += c.visits_plain;
    }
    o->gpu_seconds = S->gpu_seconds;
    o->kernel_seconds = S->kernel_seconds;
    o->kernel_launches = S->kernel_launches;
    o->time_bits = S->TB;
    o->counter_bits = S->NB;
    o->rank_bits = 0;   // the (t, c) tie-break needs no bits in the word (explicit id order)
    const int ncls = 2 * (2 * S->ndim + 1);
    double rate = 0;
    for (int k = 0; k < ncls; ++k) {
        o->class_hist[k] = S->h_stat->hist[k];
        rate += (double)S->h_stat->hist[k] * ((double)S->thr[k] / 4294967296.0);
    }
    o->nfold_rate = rate * S->lambda;
    return ACA_OK;
}

int aca_get_tile_grid(const aca_sim* S, int64_t* out) {
    if (!S || !out) return fail(ACA_EINVAL, "null argument");
    if (S->whole || S->sync || S->shards.empty()) return fail(ACA_ESTATE, "the handle runs no tile kernel");
    const Shard& sh = S->shards[0];
    out[0] = sh.tiles_x; out[1] = sh.tiles_y; out[2] = sh.tiles_z; out[3] = (int64_t)S->shards.size();
    out[4] = S->tile[0]; out[5] = S->tile[1]; out[6] = S->tile[2];
    return ACA_OK;
}

int aca_get_tile_classes(aca_sim* S, uint32_t* out, size_t count, int refresh) {
    if (!S || !out) return fail(ACA_EINVAL, "null argument");
    if (!S->cls) return fail(ACA_ESTATE, "class bookkeeping is off (aca_options.class_book = 0)");
    size_t want = 0;
    for (auto& sh : S->shards) want += (size_t)sh.tiles_x * sh.tiles_y * sh.tiles_z * 16;
    if (count != want) return fail(ACA_EINVAL, "count %zu != %zu (16 per tile)", count, want);
    CK(cudaSetDevice(S->device));
    if (refresh || S->cls_stale) {
        if (!S->ipc) {   // single process: the halos of sharded handles from the current rows
            int rc = exchange(S);
            if (rc) return rc;
        }
        int rc = class_refresh(S);
        if (rc) return rc;
    }
    size_t off = 0;
    for (auto& sh : S->shards) {
        const size_t n = (size_t)sh.tiles_x * sh.tiles_y * sh.tiles_z * 16;
        CK(cudaMemcpyAsync(out + off, sh.tile_hist, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, S->stream));
        off += n;
    }
    CK(cudaStreamSynchronize(S->stream));
    return ACA_OK;
}

int aca_set_state(aca_sim* S, const int8_t* spins, const uint64_t* times, const uint32_t* counters, size_t count) {
    int rc = check_count(S, count, spins);
    if (rc) return rc;
    S->cls_stale = true;
    if (S->ipc) S->snap_valid = false;   // the neighbours' boundary rows are unknown until a run
    if (!times || !counters) return fail(ACA_EINVAL, "null times/counters");
    CK(cudaSetDevice(S->device));
    uint64_t tmax = 0;
    uint32_t nmax = 0;
    for (size_t i = 0; i < count; ++i) {
        if (spins[i] != 1 && spins[i] != -1) return fail(ACA_EINVAL, "spin %zu is not +-1", i);
        if (times[i] < 1) return fail(ACA_ERANGE, "time %zu must be >= 1", i);
        tmax = std::max<uint64_t>(tmax, times[i]);
        nmax = std::max(nmax, counters[i]);
    }
    // layout able to hold the largest time (plus one more increment) and counter
    const int tb = bits_for(tmax + S->max_delta);
    int nb = std::min(31, 63 - tb);
    if (nb < 1 || (uint64_t)nmax >= (1ull << nb) - 1ull) return fail(ACA_ERANGE, "state does not fit the packed word");
    S->NB = nb;
    S->TB = 63 - nb;
    S->t_hi = tmax + 1;
    set_geo_layout(S);
    drop_graph(S);
    rc = ensure_scratch(S, CHUNK * 13);
    if (rc) return rc;
    unsigned long long* dt = (unsigned long long*)S->scratch;
    unsigned int* dn = (unsigned int*)(dt + CHUNK);
    int8_t* ds = (int8_t*)(dn + CHUNK);
    size_t off = 0;
    for (auto& sh : S->shards) {
        for (size_t b = 0; b < sh.n; b += CHUNK) {
            const size_t m = std::min(CHUNK, sh.n - b);
            CK(cudaMemcpyAsync(dt, times + off + b, m * 8, cudaMemcpyHostToDevice, S->stream));
            CK(cudaMemcpyAsync(dn, counters + off + b, m * 4, cudaMemcpyHostToDevice, S->stream));
            CK(cudaMemcpyAsync(ds, spins + off + b, m, cudaMemcpyHostToDevice, S->stream));
            pack_kernel<<<592, 256, 0, S->stream>>>(sh.words + b, ds, dt, dn, sh.g, (unsigned long long)m);
            CK(cudaGetLastError());
            CK(cudaStreamSynchronize(S->stream));
        }
        off += sh.n;
    }
    S->T_last = 0;
    return ACA_OK;
}

int aca_set_spins(aca_sim* S, const int8_t* spins, size_t count) {
    int rc = check_count(S, count, spins);
    if (rc) return rc;
    S->cls_stale = true;
    if (S->ipc) S->snap_valid = false;   // the neighbours' boundary rows are unknown until a run
    CK(cudaSetDevice(S->device));
    rc = ensure_scratch(S, CHUNK);
    if (rc) return rc;
    size_t off = 0;
    for (auto& sh : S->shards) {
        for (size_t b = 0; b < sh.n; b += CHUNK) {
            const size_t m = std::min(CHUNK, sh.n - b);
            CK(cudaMemcpyAsync(S->scratch, spins + off + b, m, cudaMemcpyHostToDevice, S->stream));
            pack_kernel<<<592, 256, 0, S->stream>>>(sh.words + b, (const int8_t*)S->scratch, nullptr, nullptr, sh.g,
                                                    (unsigned long long)m);
            CK(cudaGetLastError());
        }
        off += sh.n;
    }
    CK(cudaStreamSynchronize(S->stream));
    return ACA_OK;
}

// ---------------------------------------------------------------- asynchronous spin I/O
static int ensure_async_io(aca_sim* S) {
    if (S->cstream) return ACA_OK;
    size_t n = 0;
    for (auto& sh : S->shards) n += sh.n;
    CK(cudaStreamCreateWithFlags(&S->cstream, cudaStreamNonBlocking));
    for (int a = 0; a < 2; ++a) {
        if (cudaMalloc(&S->stage_in[a], n) != cudaSuccess || cudaMalloc(&S->stage_out[a], n) != cudaSuccess)
            return fail(ACA_ENOMEM, "staging buffers (%zu cells)", n);
        for (cudaEvent_t* e : {&S->ev_h2d[a], &S->ev_pack[a], &S->ev_unp[a], &S->ev_d2h[a]})
            CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        // initial state: nothing pending on any slot
        CK(cudaEventRecord(S->ev_pack[a], S->stream));
        CK(cudaEventRecord(S->ev_d2h[a], S->cstream));
    }
    return ACA_OK;
}

int aca_stage_spins(aca_sim* S, const int8_t* spins, size_t count, int slot) {
    int rc = check_count(S, count, spins);
    if (rc) return rc;
    if (slot < 0 || slot > 1) return fail(ACA_EINVAL, "slot must be 0 or 1");
    CK(cudaSetDevice(S->device));
    rc = ensure_async_io(S);
    if (rc) return rc;
    CK(cudaStreamWaitEvent(S->cstream, S->ev_pack[slot], 0));   // the slot's previous pack has read it
    CK(cudaMemcpyAsync(S->stage_in[slot], spins, count, cudaMemcpyHostToDevice, S->cstream));
    CK(cudaEventRecord(S->ev_h2d[slot], S->cstream));
    return ACA_OK;
}

int aca_set_spins_staged(aca_sim* S, int slot) {
    if (!S) return fail(ACA_EINVAL, "null handle");
    S->cls_stale = true;
    if (S->ipc) S->snap_valid = false;
    if (slot < 0 || slot > 1) return fail(ACA_EINVAL, "slot must be 0 or 1");
    if (!S->cstream) return fail(ACA_ESTATE, "nothing staged (call aca_stage_spins first)");
    CK(cudaSetDevice(S->device));
    CK(cudaStreamWaitEvent(S->stream, S->ev_h2d[slot], 0));
    size_t off = 0;
    for (auto& sh : S->shards) {
        pack_kernel<<<1184, 256, 0, S->stream>>>(sh.words, S->stage_in[slot] + off, nullptr, nullptr, sh.g,
                                                 (unsigned long long)sh.n);
        CK(cudaGetLastError());
        off += sh.n;
    }
    CK(cudaEventRecord(S->ev_pack[slot], S->stream));
    return ACA_OK;
}

int aca_get_spins_async(aca_sim* S, int8_t* out, size_t count) {
    int rc = check_count(S, count, out);
    if (rc) return rc;
    CK(cudaSetDevice(S->device));
    rc = ensure_async_io(S);
    if (rc) return rc;
    const int k = S->out_slot;
    S->out_slot ^= 1;
    CK(cudaStreamWaitEvent(S->stream, S->ev_d2h[k], 0));       // the slot's previous copy has drained
    size_t off = 0;
    for (auto& sh : S->shards) {
        unpack_kernel<<<1184, 256, 0, S->stream>>>(sh.words, S->stage_out[k] + off, nullptr, nullptr, sh.g, sh.n);
        CK(cudaGetLastError());
        off += sh.n;
    }
    CK(cudaEventRecord(S->ev_unp[k], S->stream));
    CK(cudaStreamWaitEvent(S->cstream, S->ev_unp[k], 0));
    CK(cudaMemcpyAsync(out, S->stage_out[k], count, cudaMemcpyDeviceToHost, S->cstream));
    CK(cudaEventRecord(S->ev_d2h[k], S->cstream));
    return ACA_OK;
}

int aca_sync(aca_sim* S) {
    if (!S) return fail(ACA_EINVAL, "null handle");
    CK(cudaSetDevice(S->device));
    CK(cudaStreamSynchronize(S->stream));
    if (S->cstream) CK(cudaStreamSynchronize(S->cstream));
    return ACA_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- self-test hooks
namespace {
__global__ void philox_test_kernel(uint64_t n, const uint32_t* ctr, const uint32_t* key, uint32_t* out, uint32_t* ref) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        u32x4 r = philox4x32_10(ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3], key[2 * i], key[2 * i + 1]);
        uint32_t rk[20];
        philox_round_keys(key[2 * i], key[2 * i + 1], rk);
        const u32x4 r2 = philox4x32_10_rk(ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3], rk);
        if (r2.x != r.x || r2.y != r.y || r2.z != r.z || r2.w != r.w) {   // both forms must agree
            r.x = ~r.x; r.y = ~r.y; r.z = ~r.z; r.w = ~r.w;
        }
        out[4 * i] = r.x; out[4 * i + 1] = r.y; out[4 * i + 2] = r.z; out[4 * i + 3] = r.w;
        uint4 c = make_uint4(ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]);
        uint2 k = make_uint2(key[2 * i], key[2 * i + 1]);
        const uint4 q = curand_Philox4x32_10(c, k);
        ref[4 * i] = q.x; ref[4 * i + 1] = q.y; ref[4 * i + 2] = q.z; ref[4 * i + 3] = q.w;
    }
}
// The tile kernels read the NLOG-2 tables split in shared memory (NlogSmem); the one-pass and
// aggregated kernels read the interleaved table (NlogLR). Both views must give the same integers:
// a disagreement is reported as the bitwise complement (the test then fails).
__global__ void nlog_test_kernel(uint64_t n, const uint64_t* X, uint64_t* q, uint64_t* d, const unsigned long long* lr_g,
                                 unsigned long long inv_lambda, int tie_bits) {
    __shared__ unsigned long long Lt[256];
    __shared__ unsigned int Rt[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) { Lt[i] = lr_g[2 * i]; Rt[i] = (unsigned int)lr_g[2 * i + 1]; }
    __syncthreads();
    const NlogSmem tab{smem_u32(Lt), smem_u32(Rt)};
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t a = nlog_q32_t(X[i], tab, ACA_LN2_Q48), b = nlog_q32(X[i], lr_g, ACA_LN2_Q48);
        q[i] = a == b ? a : ~a;
        const uint64_t da = delta_q32_t((uint32_t)(X[i] >> 32), (uint32_t)X[i], tab, ACA_LN2_Q48, inv_lambda, tie_bits);
        const uint64_t db = delta_q32((uint32_t)(X[i] >> 32), (uint32_t)X[i], lr_g, ACA_LN2_Q48, inv_lambda, tie_bits);
        d[i] = da == db ? da : ~da;
    }
}
__global__ void law_test_kernel(uint64_t n, const uint64_t* X, uint64_t* u, uint64_t* d, const unsigned long long* lr_g,
                                unsigned long long inv_lambda, int tie_bits, int law) {
    __shared__ unsigned long long Lt[256];
    __shared__ unsigned int Rt[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) { Lt[i] = lr_g[2 * i]; Rt[i] = (unsigned int)lr_g[2 * i + 1]; }
    __syncthreads();
    const NlogSmem tab{smem_u32(Lt), smem_u32(Rt)};
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t w1 = (uint32_t)(X[i] >> 32), w2 = (uint32_t)X[i];
        if (law == 4) {   // the period of law 4 from (w3, c_lo) = (w1, w2): gauss_u(w3, w3, c_lo, 10)
            const uint64_t ua = gauss_u(w1, w1, w2, 10u, tab, ACA_LN2_Q48), ub = gauss_u(w1, w1, w2, 10u, NlogLR{lr_g}, ACA_LN2_Q48);
            u[i] = ua == ub ? ua : ~ua;
            d[i] = delta_of_u(ua, inv_lambda, tie_bits);
            continue;
        }
        const uint64_t ua = law_q32_t(w1, w2, tab, ACA_LN2_Q48, law), ub = law_q32(w1, w2, lr_g, ACA_LN2_Q48, law);
        u[i] = ua == ub ? ua : ~ua;
        const uint64_t da = delta_q32_t(w1, w2, tab, ACA_LN2_Q48, inv_lambda, tie_bits, law);
        const uint64_t db = delta_q32(w1, w2, lr_g, ACA_LN2_Q48, inv_lambda, tie_bits, law);
        d[i] = da == db ? da : ~da;
    }
}
}  // namespace

extern "C" {
int aca_selftest_law(uint64_t n, const uint64_t* X, int law, uint64_t inv_lambda, int tie_bits, uint64_t* u,
                     uint64_t* delta) {
    if (!X || !u || !delta) return fail(ACA_EINVAL, "null buffer");
    if (law < 0 || law > 4) return fail(ACA_EINVAL, "bad law");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || !ndev) { cudaGetLastError(); return fail(ACA_ENODEV, "no CUDA device"); }
    uint64_t *dx = nullptr, *du = nullptr, *dd = nullptr;
    unsigned long long* dlr = nullptr;
    CK(cudaMalloc(&dx, n * 8)); CK(cudaMalloc(&du, n * 8)); CK(cudaMalloc(&dd, n * 8));
    CK(cudaMalloc(&dlr, sizeof(ACA_NLOG_LR)));
    CK(cudaMemcpy(dlr, ACA_NLOG_LR, sizeof(ACA_NLOG_LR), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dx, X, n * 8, cudaMemcpyHostToDevice));
    law_test_kernel<<<592, 256>>>(n, dx, du, dd, dlr, inv_lambda, tie_bits, law);
    CK(cudaGetLastError());
    CK(cudaMemcpy(u, du, n * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(delta, dd, n * 8, cudaMemcpyDeviceToHost));
    cudaFree(dx); cudaFree(du); cudaFree(dd); cudaFree(dlr);
    return ACA_OK;
}

int aca_selftest_philox(uint64_t n, const uint32_t* ctr, const uint32_t* key, uint32_t* out, uint32_t* ref) {
    if (!ctr || !key || !out || !ref) return fail(ACA_EINVAL, "null buffer");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || !ndev) { cudaGetLastError(); return fail(ACA_ENODEV, "no CUDA device"); }
    uint32_t *dc = nullptr, *dk = nullptr, *do_ = nullptr, *dr = nullptr;
    CK(cudaMalloc(&dc, n * 16)); CK(cudaMalloc(&dk, n * 8)); CK(cudaMalloc(&do_, n * 16)); CK(cudaMalloc(&dr, n * 16));
    CK(cudaMemcpy(dc, ctr, n * 16, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dk, key, n * 8, cudaMemcpyHostToDevice));
    philox_test_kernel<<<592, 256>>>(n, dc, dk, do_, dr);
    CK(cudaGetLastError());
    CK(cudaMemcpy(out, do_, n * 16, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ref, dr, n * 16, cudaMemcpyDeviceToHost));
    cudaFree(dc); cudaFree(dk); cudaFree(do_); cudaFree(dr);
    return ACA_OK;
}

int aca_selftest_nlog(uint64_t n, const uint64_t* X, uint64_t* q, uint64_t* delta, uint64_t inv_lambda, int tie_bits) {
    if (!X || !q || !delta) return fail(ACA_EINVAL, "null buffer");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || !ndev) { cudaGetLastError(); return fail(ACA_ENODEV, "no CUDA device"); }
    uint64_t *dx = nullptr, *dq = nullptr, *dd = nullptr;
    unsigned long long* dlr = nullptr;
    CK(cudaMalloc(&dx, n * 8)); CK(cudaMalloc(&dq, n * 8)); CK(cudaMalloc(&dd, n * 8));
    CK(cudaMalloc(&dlr, sizeof(ACA_NLOG_LR)));
    CK(cudaMemcpy(dlr, ACA_NLOG_LR, sizeof(ACA_NLOG_LR), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dx, X, n * 8, cudaMemcpyHostToDevice));
    nlog_test_kernel<<<592, 256>>>(n, dx, dq, dd, dlr, inv_lambda, tie_bits);
    CK(cudaGetLastError());
    CK(cudaMemcpy(q, dq, n * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(delta, dd, n * 8, cudaMemcpyDeviceToHost));
    cudaFree(dx); cudaFree(dq); cudaFree(dd); cudaFree(dlr);
    return ACA_OK;
}

// ---------------------------------------------------------------- fig:perfbl model (P11)
int aca_perfbl_run(int64_t px, int64_t py, int m, double lag, uint64_t seed, int64_t rounds, uint64_t* ups,
                   uint64_t* h_out, uint32_t* n_out, int device) {
    if (px < 1 || py < 1 || px * py > ((int64_t)1 << 24)) return fail(ACA_EINVAL, "PE grid must have 1 .. 2^24 PEs");
    if (m < 2 || m > 65535) return fail(ACA_EINVAL, "m must be in [2, 65535]");
    if (!(lag >= 0) || !std::isfinite(lag)) return fail(ACA_EINVAL, "lag must be >= 0 (0 = unbounded)");
    if (rounds < 0 || (rounds > 0 && !ups)) return fail(ACA_EINVAL, "bad rounds / null ups");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || !ndev) { cudaGetLastError(); return fail(ACA_ENODEV, "no CUDA device"); }
    if (device >= 0) CK(cudaSetDevice(device));
    const int64_t N = px * py;
    PerfblParams A{};
    A.px = (int)px; A.py = (int)py;
    const unsigned long long mm = (unsigned long long)m * (unsigned long long)m;
    A.E1 = ((unsigned long long)(m - 2) * (unsigned long long)(m - 2) << 32) / mm;
    A.E2 = ((mm - 4) << 32) / mm;
    A.lag = lag > 0 ? (unsigned long long)std::floor(lag * 4294967296.0 + 0.5) : 0ull;
    philox_round_keys((uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32), A.rk);
    A.rounds = rounds;
    unsigned long long* dlr = nullptr;
    CK(cudaMalloc(&A.hb, (size_t)N * 16));
    CK(cudaMalloc(&A.n, (size_t)N * 4));
    CK(cudaMalloc(&A.ups, (size_t)(rounds > 0 ? rounds : 1) * 8));
    CK(cudaMalloc(&dlr, sizeof(ACA_NLOG_LR)));
    CK(cudaMemcpy(dlr, ACA_NLOG_LR, sizeof(ACA_NLOG_LR), cudaMemcpyHostToDevice));
    perfbl_kernel<1024><<<1, 1024>>>(A, dlr);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    if (rounds > 0) CK(cudaMemcpy(ups, A.ups, (size_t)rounds * 8, cudaMemcpyDeviceToHost));
    if (h_out) CK(cudaMemcpy(h_out, A.hb + (size_t)(rounds & 1) * N, (size_t)N * 8, cudaMemcpyDeviceToHost));
    if (n_out) CK(cudaMemcpy(n_out, A.n, (size_t)N * 4, cudaMemcpyDeviceToHost));
    cudaFree(A.hb); cudaFree(A.n); cudaFree(A.ups); cudaFree(dlr);
    return ACA_OK;
}

// ---------------------------------------------------------------- time-only efficiency model
int aca_efficiency_run(int ndim, const int64_t* dims, int law, double lambda, uint64_t seed, int64_t rounds,
                       uint64_t* fired_per_round, uint64_t* t_out, int device, double* gpu_seconds) {
    return aca_efficiency_run_q(ndim, dims, law, lambda, seed, rounds, 1, fired_per_round, t_out, device, gpu_seconds);
}

int aca_efficiency_run_q(int ndim, const int64_t* dims, int law, double lambda, uint64_t seed, int64_t rounds, int q,
                         uint64_t* fired_per_round, uint64_t* t_out, int device, double* gpu_seconds) {
    if (ndim < 1 || ndim > 3 || !dims) return fail(ACA_EINVAL, "ndim must be 1, 2 or 3");
    if (q < 1 || q > 8) return fail(ACA_EINVAL, "q must be in [1, 8]");
    if (law < 0 || law > 3) return fail(ACA_EINVAL, "law must be 0, 1, 2 or 3");
    if (!(lambda > 0) || !std::isfinite(lambda)) return fail(ACA_EINVAL, "lambda must be > 0");
    if (rounds < 0 || rounds > (int64_t)1 << 31) return fail(ACA_EINVAL, "rounds out of range");
    if (rounds > 0 && !fired_per_round) return fail(ACA_EINVAL, "null fired_per_round");
    int64_t N = 1;
    for (int a = 0; a < ndim; ++a) {
        if (dims[a] < 2) return fail(ACA_EINVAL, "every dimension must be >= 2");
        N *= dims[a];
        if (N > (int64_t)1 << 34) return fail(ACA_EINVAL, "lattice too large");
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || !ndev) { cudaGetLastError(); return fail(ACA_ENODEV, "no CUDA device"); }
    if (device >= 0) CK(cudaSetDevice(device));
    EffParams P{};
    P.ndim = ndim;
    P.nx = dims[0]; P.ny = ndim >= 2 ? dims[1] : 1; P.nz = ndim == 3 ? dims[2] : 1; P.N = N;
    philox_round_keys((uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32), P.rk);
    P.inv_lambda = (unsigned long long)std::floor(4294967296.0 / lambda + 0.5);
    P.law = law;
    P.q = q;
    const bool small = N < ((int64_t)1 << 32) && q == 1;   // 32-bit indices: Lemire division, compacted kernel
    bool stream2d = true;                                   // 2-D row-streaming kernel (ACA_EFF_STREAM=0: off)
    if (const char* e = getenv("ACA_EFF_STREAM")) stream2d = atoi(e) != 0;
    auto recip = [](unsigned long long d) { return (unsigned long long)(~0ull / d) + 1ull; };   // ceil(2^64/d), d >= 2
    P.mx = recip((unsigned long long)P.nx);
    P.my = recip((unsigned long long)P.ny < 2 ? 2ull : (unsigned long long)P.ny);
    unsigned long long *a = nullptr, *b = nullptr, *fired = nullptr, *dlr = nullptr;
    cudaStream_t st = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    auto cleanup = [&]() {
        if (st) cudaStreamSynchronize(st);
        cudaFree(a); cudaFree(b); cudaFree(fired); cudaFree(dlr);
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
        if (st) cudaStreamDestroy(st);
    };
    if (cudaMalloc(&a, (size_t)N * 8) != cudaSuccess || cudaMalloc(&b, (size_t)N * 8) != cudaSuccess ||
        cudaMalloc(&fired, (size_t)std::max<int64_t>(rounds, 1) * 8) != cudaSuccess ||
        cudaMalloc(&dlr, sizeof(ACA_NLOG_LR)) != cudaSuccess) {
        cleanup();
        return fail(ACA_ENOMEM, "device allocation failed (%lld cells)", (long long)N);
    }
    int rc = ACA_OK;
    do {
        if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) { rc = fail(ACA_ECUDA, "stream"); break; }
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaMemcpyAsync(dlr, ACA_NLOG_LR, sizeof(ACA_NLOG_LR), cudaMemcpyHostToDevice, st);
        cudaMemsetAsync(fired, 0, (size_t)std::max<int64_t>(rounds, 1) * 8, st);
        int nsm = 148;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device >= 0 ? device : 0);
        const long long want = (N + 255) / 256;
        const unsigned grid = (unsigned)std::min<long long>(want, (long long)nsm * 8);
        eff_init_kernel<<<grid, 256, 0, st>>>(a, P, dlr);
        cudaEventRecord(e0, st);
        for (int64_t r = 0; r < rounds; ++r) {
            const unsigned long long* tin = (r & 1) ? b : a;
            unsigned long long* tout = (r & 1) ? a : b;
            if (small && ndim == 2 && stream2d) {
                const dim3 g2((unsigned)((P.nx + EFF_W - 1) / EFF_W), (unsigned)((P.ny + EFF_H - 1) / EFF_H));
                eff_round_kernel_2d<<<g2, EFF_W, 0, st>>>(tin, tout, P, dlr, (uint32_t)r, fired);
            } else if (small) {
                if (ndim == 1) eff_round_kernel_c<1><<<grid, 256, 0, st>>>(tin, tout, P, dlr, (uint32_t)r, fired);
                else if (ndim == 2) eff_round_kernel_c<2><<<grid, 256, 0, st>>>(tin, tout, P, dlr, (uint32_t)r, fired);
                else eff_round_kernel_c<3><<<grid, 256, 0, st>>>(tin, tout, P, dlr, (uint32_t)r, fired);
            } else if (ndim == 1) eff_round_kernel<1><<<grid, 256, 0, st>>>(tin, tout, P, dlr, (uint32_t)r, fired);
            else if (ndim == 2) eff_round_kernel<2><<<grid, 256, 0, st>>>(tin, tout, P, dlr, (uint32_t)r, fired);
            else eff_round_kernel<3><<<grid, 256, 0, st>>>(tin, tout, P, dlr, (uint32_t)r, fired);
        }
        cudaEventRecord(e1, st);
        if (cudaStreamSynchronize(st) != cudaSuccess || cudaGetLastError() != cudaSuccess) {
            rc = fail(ACA_ECUDA, "efficiency kernels failed");
            break;
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (gpu_seconds) *gpu_seconds = ms * 1e-3;
        if (rounds > 0 && cudaMemcpy(fired_per_round, fired, (size_t)rounds * 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
            rc = fail(ACA_ECUDA, "copy counts");
            break;
        }
        if (t_out && cudaMemcpy(t_out, (rounds & 1) ? b : a, (size_t)N * 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
            rc = fail(ACA_ECUDA, "copy times");
            break;
        }
    } while (0);
    cleanup();
    return rc;
}

// ---------------------------------------------------------------- output frames (fig:genout)
int aca_run_frames(aca_sim* S, double dt, int64_t K0, int64_t count, int B, uint8_t* out) {
    if (!S || !out) return fail(ACA_EINVAL, "null argument");
    if (!(dt > 0) || !std::isfinite(dt)) return fail(ACA_EINVAL, "dt must be > 0");
    if (K0 < 0 || count < 1) return fail(ACA_EINVAL, "K0 >= 0 and count >= 1 required");
    if (B < 1 || B > 16) return fail(ACA_EINVAL, "B must be in [1, 16]");
    const double dq = std::floor(dt * 4294967296.0 + 0.5);
    if (dq < 1 || dq * (double)(K0 + count) >= 1.8e19) return fail(ACA_ERANGE, "frame times overflow");
    const unsigned long long dtq = (unsigned long long)dq;
    if (S->T_last > (unsigned long long)K0 * dtq + 1ull)
        return fail(ACA_ESTATE, "frame K0 lies before the time already simulated");
    CK(cudaSetDevice(S->device));
    size_t nloc = 0;
    for (auto& sh : S->shards) nloc += sh.n;
    const size_t wpf = (nloc + 31) / 32;
    const size_t need = (size_t)B * wpf * 4;
    if (S->frame_ring_bytes < need) {
        cudaFree(S->frame_ring);
        S->frame_ring = nullptr;
        S->frame_ring_bytes = 0;
        CK(cudaMalloc(&S->frame_ring, need));
        S->frame_ring_bytes = need;
    }
    const size_t fbytes = (nloc + 7) / 8;
    const long long base = S->world > 1 ? (long long)(S->shards[0].g.ndim == 2
                                                          ? (long long)S->shards[0].g.y0 * S->shards[0].g.nx
                                                          : (long long)S->shards[0].g.z0 * S->shards[0].g.ny * S->shards[0].g.nx)
                                        : 0;
    int rc = ACA_OK;
    for (int64_t K = K0; K < K0 + count && rc == ACA_OK; ) {
        const int nb = (int)std::min<int64_t>(B, K0 + count - K);
        CK(cudaMemsetAsync(S->frame_ring, 0, (size_t)nb * wpf * 4, S->stream));
        S->fr.bits = S->frame_ring;
        S->fr.t0 = (unsigned long long)K * dtq;
        S->fr.dt = dtq;
        S->fr.wpf = wpf;
        S->fr.base = base;
        S->fr.nb = nb;
        drop_graph(S);   // kernel parameters changed
        unsigned long long off = 0;
        for (auto& sh : S->shards) {
            frame_prefill_kernel<<<592, 256, 0, S->stream>>>(sh.words, sh.g, S->fr, (unsigned long long)sh.n, off);
            CK(cudaGetLastError());
            off += sh.n;
        }
        rc = aca_run_until_q32(S, (unsigned long long)(K + nb - 1) * dtq + 1ull);
        if (rc == ACA_OK) {
            for (int k = 0; k < nb; ++k)
                CK(cudaMemcpyAsync(out + (size_t)(K - K0 + k) * fbytes, S->frame_ring + (size_t)k * wpf, fbytes,
                                   cudaMemcpyDeviceToHost, S->stream));
            CK(cudaStreamSynchronize(S->stream));
        }
        K += nb;
    }
    S->fr = FrameParams{};
    drop_graph(S);
    return rc;
}

// ---------------------------------------------------------------- aggregated Poisson stream
static int agg_run_impl(bool bkl, const int64_t* dims, int m, double lambda, double beta, double J, double h, int rule,
                        uint64_t seed, double init_q, double T, int budget, int8_t* spins_out, uint64_t* T_out,
                        uint32_t* n_out, aca_agg_stats* st, int device) {
    if (!dims) return fail(ACA_EINVAL, "null dims");
    if (m < 1 || m > 32) return fail(ACA_EINVAL, "m must be in [1, 32]");
    if (bkl && m == 1) return fail(ACA_EINVAL, "modified BKL needs m >= 2");
    if (bkl && !(lambda >= 1e-6)) return fail(ACA_EINVAL, "modified BKL needs lambda >= 1e-6");
    const int64_t nx = dims[0], ny = dims[1];
    if (nx < 2 || ny < 2 || nx % m || ny % m || nx * ny > ((int64_t)1 << 32) || nx > (1 << 30) || ny > (1 << 30))
        return fail(ACA_EINVAL, "dims must be >= 2, multiples of m, N <= 2^32");
    if (!(lambda > 0) || !std::isfinite(lambda) || !(beta >= 0) || !std::isfinite(beta) || !std::isfinite(J) ||
        !std::isfinite(h))
        return fail(ACA_EINVAL, "bad lambda / beta / J / h");
    if (rule != ACA_HEATBATH && rule != ACA_METROPOLIS) return fail(ACA_EINVAL, "rule must be 0 or 1");
    if (!(init_q >= 0 && init_q <= 1)) return fail(ACA_EINVAL, "init_q must be in [0, 1]");
    if (!(T >= 0) || !std::isfinite(T) || T * 4294967296.0 > 1.8e19) return fail(ACA_EINVAL, "bad T");
    if (budget < 1) budget = 64;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || !ndev) { cudaGetLastError(); return fail(ACA_ENODEV, "no CUDA device"); }
    if (device >= 0) CK(cudaSetDevice(device));
    AggParams A{};
    A.nx = (int)nx; A.ny = (int)ny; A.m = m;
    A.mx = (int)(nx / m); A.my = (int)(ny / m);
    philox_round_keys((uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32), A.rk);
    A.inv = (unsigned long long)std::floor(4294967296.0 / (lambda * (double)(m * m)) + 0.5);
    A.Tend = (unsigned long long)std::floor(T * 4294967296.0 + 0.5);
    A.tag_e = m == 1 ? 0u : 3u;
    A.tag_i = m == 1 ? 1u : 4u;
    A.budget = budget;
    A.do_hash = 1;
    unsigned long long thr[14];
    flip_table(2, beta, J, h, rule, thr);
    for (int i = 0; i < 10; ++i) A.thr[i] = thr[i];
    A.thr_init = (unsigned long long)std::floor(init_q * 4294967296.0);
    BklExtra E{};
    E.lambda = lambda;
    E.kcol = m > 2 ? (((1u << (m - 1)) - 1u) & ~1u) : 0u;   // columns 1 .. m - 2
    E.W0 = (unsigned long long)(4 * m - 4) << 32;
    const int64_t NC = (int64_t)A.mx * A.my;
    unsigned long long* dlr = nullptr;
    AggAcc* dacc = nullptr;
    int8_t* dsp = nullptr;
    cudaStream_t str = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    auto cleanup = [&]() {
        if (str) cudaStreamSynchronize(str);
        cudaFree(A.rows); cudaFree(A.T); cudaFree(A.n); cudaFree(dlr); cudaFree(dacc); cudaFree(dsp);
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
        if (str) cudaStreamDestroy(str);
    };
    if (cudaMalloc(&A.rows, (size_t)NC * m * 4) != cudaSuccess || cudaMalloc(&A.T, NC * 8) != cudaSuccess ||
        cudaMalloc(&A.n, NC * 4) != cudaSuccess || cudaMalloc(&dlr, sizeof(ACA_NLOG_LR)) != cudaSuccess ||
        cudaMalloc(&dacc, sizeof(AggAcc)) != cudaSuccess) {
        cleanup();
        return fail(ACA_ENOMEM, "device allocation failed");
    }
    int rc = ACA_OK;
    AggAcc hacc{};
    uint64_t launches = 0;
    do {
        if (cudaStreamCreateWithFlags(&str, cudaStreamNonBlocking) != cudaSuccess) { rc = fail(ACA_ECUDA, "stream"); break; }
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaMemcpyAsync(dlr, ACA_NLOG_LR, sizeof(ACA_NLOG_LR), cudaMemcpyHostToDevice, str);
        cudaMemsetAsync(dacc, 0, sizeof(AggAcc), str);
        int nsm = 148;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device >= 0 ? device : 0);
        const unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>((NC + 255) / 256, (long long)nsm * 8));
        if (bkl) bkl_init_kernel<<<grid, 256, 0, str>>>(A, E, dlr);
        else agg_init_kernel<<<grid, 256, 0, str>>>(A, dlr);
        cudaEventRecord(e0, str);
        for (int batch = 0;; ++batch) {
            for (int kk = 0; kk < 8; ++kk) {
                if (kk == 7) cudaMemsetAsync(&dacc->active, 0, 16, str);   // active + blocked of the last launch
                if (bkl) bkl_round_kernel<<<grid, 256, 0, str>>>(A, E, dlr, dacc);
                else agg_round_kernel<<<grid, 256, 0, str>>>(A, dlr, dacc);
                ++launches;
            }
            if (cudaMemcpyAsync(&hacc, dacc, sizeof(AggAcc), cudaMemcpyDeviceToHost, str) != cudaSuccess ||
                cudaStreamSynchronize(str) != cudaSuccess) {
                rc = fail(ACA_ECUDA, "aggregated kernels failed: %s", cudaGetErrorString(cudaGetLastError()));
                break;
            }
            if (hacc.active == 0) break;
            if (batch > (1 << 24)) { rc = fail(ACA_ESTATE, "no termination"); break; }
        }
        if (rc) break;
        cudaEventRecord(e1, str);
        cudaStreamSynchronize(str);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (spins_out) {
            if (cudaMalloc(&dsp, (size_t)nx * ny) != cudaSuccess) { rc = fail(ACA_ENOMEM, "spins"); break; }
            agg_unpack_kernel<<<grid, 256, 0, str>>>(A, dsp);
            if (cudaMemcpyAsync(spins_out, dsp, (size_t)nx * ny, cudaMemcpyDeviceToHost, str) != cudaSuccess) {
                rc = fail(ACA_ECUDA, "copy spins");
                break;
            }
        }
        if (T_out && cudaMemcpyAsync(T_out, A.T, NC * 8, cudaMemcpyDeviceToHost, str) != cudaSuccess) { rc = fail(ACA_ECUDA, "copy T"); break; }
        if (n_out && cudaMemcpyAsync(n_out, A.n, NC * 4, cudaMemcpyDeviceToHost, str) != cudaSuccess) { rc = fail(ACA_ECUDA, "copy n"); break; }
        cudaStreamSynchronize(str);
        if (st) {
            memset(st, 0, sizeof *st);
            st->arrivals = hacc.arrivals;
            st->flips = hacc.flips;
            st->event_hash = hacc.hash;
            st->launches = launches;
            st->gpu_seconds = ms * 1e-3;
            if (spins_out) {
                long long B = 0, M = 0;
                for (int64_t y = 0; y < ny; ++y)
                    for (int64_t x = 0; x < nx; ++x) {
                        const int v = spins_out[y * nx + x];
                        M += v;
                        B += v * (spins_out[y * nx + (x + 1) % nx] + spins_out[((y + 1) % ny) * nx + x]);
                    }
                st->bond_sum = B;
                st->magnetisation = M;
            }
        }
    } while (0);
    cleanup();
    return rc;
}

int aca_agg_run(const int64_t* dims, int m, double lambda, double beta, double J, double h, int rule, uint64_t seed,
                double init_q, double T, int budget, int8_t* spins_out, uint64_t* T_out, uint32_t* n_out,
                aca_agg_stats* st, int device) {
    return agg_run_impl(false, dims, m, lambda, beta, J, h, rule, seed, init_q, T, budget, spins_out, T_out, n_out, st,
                        device);
}

int aca_bkl_run(const int64_t* dims, int m, double lambda, double beta, double J, double h, int rule, uint64_t seed,
                double init_q, double T, int budget, int8_t* spins_out, uint64_t* T_out, uint32_t* n_out,
                aca_agg_stats* st, int device) {
    return agg_run_impl(true, dims, m, lambda, beta, J, h, rule, seed, init_q, T, budget, spins_out, T_out, n_out, st,
                        device);
}

// ---------------------------------------------------------------- q-th degree neighbourhood (P12)
int aca_qnbr_run(int ndim, const int64_t* dims, int q, double lambda, double beta, double J, double h, int rule,
                 uint64_t seed, double init_q, int tie_bits, int law, double T, int rounds, int8_t* spins_out,
                 uint64_t* t_out, uint32_t* n_out, aca_qnbr_stats* st, int device) {
    if (!dims) return fail(ACA_EINVAL, "null dims");
    if (ndim != 2 && ndim != 3) return fail(ACA_EINVAL, "ndim must be 2 or 3");
    if (q < 1 || q > 4) return fail(ACA_EINVAL, "q must be in [1, 4]");
    long long N = 1;
    for (int a = 0; a < ndim; ++a) {
        if (dims[a] < 2 * q + 1 || dims[a] > (1 << 30)) return fail(ACA_EINVAL, "every side must be >= 2q + 1");
        N *= dims[a];
    }
    if (N > ((long long)1 << 32)) return fail(ACA_EINVAL, "N must be <= 2^32");
    if (!(lambda > 0) || !std::isfinite(lambda) || !(beta >= 0) || !std::isfinite(beta) || !std::isfinite(J) ||
        !std::isfinite(h))
        return fail(ACA_EINVAL, "bad lambda / beta / J / h");
    if (rule != ACA_HEATBATH && rule != ACA_METROPOLIS) return fail(ACA_EINVAL, "rule must be 0 or 1");
    if (law < 0 || law > 3) return fail(ACA_EINVAL, "law must be in [0, 3]");
    if (tie_bits < 0 || tie_bits > 40) return fail(ACA_EINVAL, "tie_bits must be in [0, 40]");
    if (!(init_q >= 0 && init_q <= 1)) return fail(ACA_EINVAL, "init_q must be in [0, 1]");
    if (!(T >= 0) || !std::isfinite(T) || T * 4294967296.0 > 1.8e19) return fail(ACA_EINVAL, "bad T");
    if (rounds < 1) rounds = 32;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || !ndev) { cudaGetLastError(); return fail(ACA_ENODEV, "no CUDA device"); }
    if (device >= 0) CK(cudaSetDevice(device));
    QParams P{};
    P.ndim = ndim; P.q = q; P.R = rounds; P.tie_bits = tie_bits; P.law = law;
    // neighbors^q(c) \ {c} = the L1 ball of radius q (closed form; the oracle builds Eq. neiq literally)
    std::vector<int> ofs;
    for (int dz = ndim == 3 ? -q : 0; dz <= (ndim == 3 ? q : 0); ++dz)
        for (int dy = -q; dy <= q; ++dy)
            for (int dx = -q; dx <= q; ++dx) {
                const int l1 = std::abs(dx) + std::abs(dy) + std::abs(dz);
                if (l1 == 0 || l1 > q) continue;
                ofs.push_back(dx); ofs.push_back(dy); ofs.push_back(dz);
            }
    P.nofs = (int)ofs.size() / 3;
    std::vector<unsigned long long> thr(2 * (P.nofs + 1));
    flip_table_z(P.nofs, beta, J, h, rule, thr.data());
    const int blk[3] = {ndim == 3 ? 8 : 32, ndim == 3 ? 8 : 32, 8};
    int ncolour = 1;
    for (int a = 0; a < 3; ++a) {
        if (a >= ndim) { P.dim[a] = 1; P.ntl[a] = 1; P.ncol[a] = 1; P.tmax[a] = 1; continue; }
        P.dim[a] = (int)dims[a];
        P.ntl[a] = std::max(2, P.dim[a] / blk[a]);
        P.ncol[a] = P.ntl[a] % 2 ? 3 : 2;
        P.tmax[a] = (P.dim[a] + P.ntl[a] - 1) / P.ntl[a];
        ncolour *= P.ncol[a];
    }
    const size_t nreg = (size_t)(P.tmax[0] + 2 * q) * (P.tmax[1] + 2 * q) * (ndim == 3 ? P.tmax[2] + 2 * q : 1);
    const size_t nimax = (size_t)P.tmax[0] * P.tmax[1] * P.tmax[2];
    const size_t smem = nreg * 9 + nimax * 13;
    if (smem > 200 * 1024) return fail(ACA_EINVAL, "tile too large for shared memory (%zu B)", smem);
    philox_round_keys((uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32), P.rk);
    P.inv = (unsigned long long)std::floor(4294967296.0 / lambda + 0.5);
    P.Tend = (unsigned long long)std::floor(T * 4294967296.0 + 0.5);
    P.thr_init = (unsigned long long)std::floor(init_q * 4294967296.0);
    unsigned long long* dlr = nullptr;
    QAcc* dacc = nullptr;
    int* dofs = nullptr;
    unsigned long long* dthr = nullptr;
    cudaStream_t str = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    auto cleanup = [&]() {
        if (str) cudaStreamSynchronize(str);
        cudaFree(P.t); cudaFree(P.s); cudaFree(P.n); cudaFree(dlr); cudaFree(dacc); cudaFree(dofs); cudaFree(dthr);
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
        if (str) cudaStreamDestroy(str);
    };
    if (cudaMalloc(&P.t, (size_t)N * 8) != cudaSuccess || cudaMalloc(&P.s, (size_t)N) != cudaSuccess ||
        cudaMalloc(&P.n, (size_t)N * 4) != cudaSuccess || cudaMalloc(&dlr, sizeof(ACA_NLOG_LR)) != cudaSuccess ||
        cudaMalloc(&dacc, sizeof(QAcc)) != cudaSuccess || cudaMalloc(&dofs, ofs.size() * sizeof(int)) != cudaSuccess ||
        cudaMalloc(&dthr, thr.size() * 8) != cudaSuccess) {
        cudaGetLastError();
        cleanup();
        return fail(ACA_ENOMEM, "device allocation failed");
    }
    P.ofs = dofs;
    P.thr = dthr;
    int rc = ACA_OK;
    QAcc hacc{};
    uint64_t launches = 0, sweeps = 0;
    do {
        if (cudaStreamCreateWithFlags(&str, cudaStreamNonBlocking) != cudaSuccess) { rc = fail(ACA_ECUDA, "stream"); break; }
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        if (cudaFuncSetAttribute(qn_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
            rc = fail(ACA_ECUDA, "shared memory attribute: %s", cudaGetErrorString(cudaGetLastError()));
            break;
        }
        cudaMemcpyAsync(dlr, ACA_NLOG_LR, sizeof(ACA_NLOG_LR), cudaMemcpyHostToDevice, str);
        cudaMemcpyAsync(dofs, ofs.data(), ofs.size() * sizeof(int), cudaMemcpyHostToDevice, str);
        cudaMemcpyAsync(dthr, thr.data(), thr.size() * 8, cudaMemcpyHostToDevice, str);
        cudaMemsetAsync(dacc, 0, sizeof(QAcc), str);
        int nsm = 148;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device >= 0 ? device : 0);
        const unsigned igrid = (unsigned)std::max<long long>(1, std::min<long long>((N + 255) / 256, (long long)nsm * 8));
        qn_init_kernel<<<igrid, 256, 0, str>>>(P, dlr);
        cudaEventRecord(e0, str);
        std::vector<unsigned> grid(ncolour);
        for (int col = 0; col < ncolour; ++col) {
            const int cc[3] = {col % P.ncol[0], (col / P.ncol[0]) % P.ncol[1], col / (P.ncol[0] * P.ncol[1])};
            unsigned g = 1;
            for (int a = 0; a < ndim; ++a)
                g *= cc[a] == 2 ? 1u : (unsigned)((P.ncol[a] == 3 ? P.ntl[a] - cc[a] : P.ntl[a] - cc[a] + 1) / 2);
            grid[col] = g;
        }
        for (int batch = 0;; ++batch) {
            for (int kk = 0; kk < 4; ++kk) {
                if (kk == 3) cudaMemsetAsync(&dacc->active, 0, 8, str);
                for (int col = 0; col < ncolour; ++col) {
                    P.colour = col;
                    qn_tile_kernel<<<grid[col], QN_THREADS, smem, str>>>(P, dlr, dacc);
                    ++launches;
                }
                ++sweeps;
            }
            if (cudaMemcpyAsync(&hacc, dacc, sizeof(QAcc), cudaMemcpyDeviceToHost, str) != cudaSuccess ||
                cudaStreamSynchronize(str) != cudaSuccess) {
                rc = fail(ACA_ECUDA, "q-neighbourhood kernels failed: %s", cudaGetErrorString(cudaGetLastError()));
                break;
            }
            if (hacc.active == 0) break;
            if (batch > (1 << 24)) { rc = fail(ACA_ESTATE, "no termination"); break; }
        }
        if (rc) break;
        cudaEventRecord(e1, str);
        qn_stats_kernel<<<igrid, QN_THREADS, 0, str>>>(P, dacc);
        if (cudaMemcpyAsync(&hacc, dacc, sizeof(QAcc), cudaMemcpyDeviceToHost, str) != cudaSuccess ||
            (spins_out && cudaMemcpyAsync(spins_out, P.s, (size_t)N, cudaMemcpyDeviceToHost, str) != cudaSuccess) ||
            (t_out && cudaMemcpyAsync(t_out, P.t, (size_t)N * 8, cudaMemcpyDeviceToHost, str) != cudaSuccess) ||
            (n_out && cudaMemcpyAsync(n_out, P.n, (size_t)N * 4, cudaMemcpyDeviceToHost, str) != cudaSuccess) ||
            cudaStreamSynchronize(str) != cudaSuccess) {
            rc = fail(ACA_ECUDA, "copy out: %s", cudaGetErrorString(cudaGetLastError()));
            break;
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (st) {
            memset(st, 0, sizeof *st);
            st->arrivals = hacc.arrivals;
            st->flips = hacc.flips;
            st->event_hash = hacc.hash;
            st->bond_sum = hacc.B2 / 2;
            st->magnetisation = hacc.M;
            st->launches = launches;
            st->sweeps = sweeps;
            st->gpu_seconds = ms * 1e-3;
        }
    } while (0);
    cleanup();
    return rc;
}

// ---------------------------------------------------------------- multi-process push (CUDA IPC)
int aca_ipc_export(const aca_sim* S, void* out, size_t size) {
    if (!S || !out) return fail(ACA_EINVAL, "null argument");
    if (!S->ipc) return fail(ACA_ESTATE, "not a multi-process push-mode handle (world > 1, halo_mode 0)");
    if (size != ACA_IPC_BLOB_BYTES) return fail(ACA_EINVAL, "blob size must be %d", ACA_IPC_BLOB_BYTES);
    CK(cudaSetDevice(S->device));
    cudaIpcMemHandle_t h[3];
    CK(cudaIpcGetMemHandle(&h[0], S->shards[0].halo_lo));
    CK(cudaIpcGetMemHandle(&h[1], S->shards[0].halo_hi));
    CK(cudaIpcGetMemHandle(&h[2], S->d_slot));
    memcpy(out, h, sizeof h);
    return ACA_OK;
}

int aca_ipc_import(aca_sim* S, const void* blobs, size_t size) {
    if (!S || !blobs) return fail(ACA_EINVAL, "null argument");
    if (!S->ipc) return fail(ACA_ESTATE, "not a multi-process push-mode handle (world > 1, halo_mode 0)");
    if (size != (size_t)S->world * ACA_IPC_BLOB_BYTES) return fail(ACA_EINVAL, "expected world x %d bytes", ACA_IPC_BLOB_BYTES);
    if (S->ipc_ready) return fail(ACA_ESTATE, "already imported");
    CK(cudaSetDevice(S->device));
    const cudaIpcMemHandle_t* H = (const cudaIpcMemHandle_t*)blobs;   // [rank][3]
    auto open = [&](int r, int which, void** p) -> int {
        if (r == S->rank) {   // own buffers (world 1 never gets here)
            *p = which == 0 ? (void*)S->shards[0].halo_lo : which == 1 ? (void*)S->shards[0].halo_hi : (void*)S->d_slot;
            return ACA_OK;
        }
        cudaError_t e = cudaIpcOpenMemHandle(p, H[3 * r + which], cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) return fail(ACA_ECUDA, "cudaIpcOpenMemHandle(rank %d): %s", r, cudaGetErrorString(e));
        S->ipc_opened.push_back(*p);
        return ACA_OK;
    };
    const int lo = (S->rank + S->world - 1) % S->world, hi = (S->rank + 1) % S->world;
    void* p = nullptr;
    int rc = open(lo, 1, &p);   // the lower neighbour's halo_hi receives my first row
    if (rc) return rc;
    S->shards[0].push_lo = (unsigned long long*)p;
    rc = open(hi, 0, &p);        // the upper neighbour's halo_lo receives my last row
    if (rc) return rc;
    S->shards[0].push_hi = (unsigned long long*)p;
    S->peer_slot.assign(S->world, nullptr);
    for (int r = 0; r < S->world; ++r) {
        rc = open(r, 2, &p);
        if (rc) return rc;
        S->peer_slot[r] = (unsigned long long*)p;
    }
    S->ipc_ready = true;
    drop_graph(S);   // kernel parameters (push pointers) changed
    return ACA_OK;
}
}  // extern "C"
