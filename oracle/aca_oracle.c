/* aca_oracle.c — serial CPU oracle. ORACLE / TEST INFRASTRUCTURE ONLY (see aca_oracle.h).
 *
 * Plain, slow, obviously correct: every arrival is processed in increasing (t, c) order
 * popped from a binary heap (global priority queue on t(c)). Each function cites the
 * passage it follows; the primitives follow docs/PRIMITIVES.md, which states the readings
 * taken where the paper is silent (generator, integer -ln, tie-break).
 * Compiled with plain gcc -O2, no fast-math (the P4 table depends on glibc exp).
 */
#include "aca_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "nlog_tables.h"
#include "gauss_tables.h"

#define ORACLE_MAXZ 128   /* the most neighbours: 3-D, q = 4 */

/* ---------------------------------------------------------------- P1: Philox4x32-10 */
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; r++) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        if (r < 9) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* ---------------------------------------------------------------- P3: NLOG-2 */
uint64_t oracle_nlog_q32(uint64_t X) {
    uint64_t x = X | 1u;
    int z = __builtin_clzll(x);
    uint64_t y = x << z;
    uint64_t m = y << 1;
    uint64_t i = m >> 56;
    uint64_t g = (m >> 24) & 0xffffffffu;
    uint64_t V = (g * ORACLE_NLOG_R[i]) >> 32;
    uint64_t V2 = V * V;
    uint64_t A = V << 8;
    uint64_t B = (V2 >> 33) + ((V2 & ((1ULL << 33) - 1)) != 0);
    uint64_t C = ((V2 >> 32) * V) / (3ULL << 40);
    uint64_t Wq = (V2 >> 32) + ((V2 & 0xffffffffULL) != 0);
    uint64_t W2 = Wq * Wq;
    uint64_t D = (W2 >> 50) + ((W2 & ((1ULL << 50) - 1)) != 0);
    uint64_t lnf = ORACLE_NLOG_L[i] + A - B + C - D;
    uint64_t S = (uint64_t)(z + 1) * ORACLE_LN2_Q48 - lnf;
    return (S + (1ULL << 15)) >> 16;
}

uint64_t oracle_inv_lambda(double lambda) { return (uint64_t)floor(4294967296.0 / lambda + 0.5); }

/* P3L: the asynchrony law, the unscaled increment U in Q32 (docs/PRIMITIVES.md P3L):
 *   law 0, Poisson (Eq. newt1i):        U = NLOG-2((w1 << 32) | w2) = -ln(r)
 *   law 1, uniform on (0,1):         U = w1
 *   law 2, next_t - t = r^(1/8):     U = floor(sqrt(sqrt(sqrt(r))) * 2^32),
 *          r = (w1 + 0.5) * 2^-32 in IEEE double (sqrt is correctly rounded). */
/* The standard normal quantile z = Phi^{-1}((w + 1/2) 2^-32) of P3L laws 3 and 4: by symmetry on
 * p' = min(p, 1 - p), s = sqrt(-ln p') with -ln p' from NLOG-2 (exact integers), |z| = G(s) by the
 * cubic pieces of oracle/gauss_tables.h (Horner in IEEE double, in this order, no fused ops). */
double oracle_gauss_z(uint32_t w) {
    const uint32_t wp = w < 0x80000000u ? w : 0xffffffffu - w;
    const uint64_t q = oracle_nlog_q32(((uint64_t)(2ull * wp + 1ull)) << 31);   /* -ln p' in Q32 */
    const double s = sqrt((double)q * (1.0 / 4294967296.0));
    const double u = (s - 0.828125) * 256.0;
    int i = (int)u;
    if (i < 0) i = 0;
    if (i > 1023) i = 1023;
    const double t = u - (double)i;
    const double* c = ORACLE_GAUSS_C[i];
    const double g = ((c[3] * t + c[2]) * t + c[1]) * t + c[0];
    return w < 0x80000000u ? -g : g;
}

/* A Gaussian period of mean 1 and standard deviation 1/4 in Q32: U = floor((1 + z/4) 2^32) for the
 * uniform word w; a period below one unit is rejected and redrawn from the sub-draws a0 of
 * Philox ctr (sa, sb, j, tag), j = 1..31, under the fixed key (0x243F6A88, 0x85A308D3); U = 1 if all
 * 32 draws fail. */
uint64_t oracle_gauss_u(uint32_t w, uint32_t sa, uint32_t sb, uint32_t tag) {
    const uint32_t kg[2] = {0x243F6A88u, 0x85A308D3u};
    for (uint32_t j = 0;; j++) {
        const double x = (1.0 + 0.25 * oracle_gauss_z(w)) * 4294967296.0;
        if (x >= 1.0) return (uint64_t)floor(x);
        if (j == 31) return 1;
        uint32_t ctr[4] = {sa, sb, j + 1, tag}, o[4];
        oracle_philox4x32_10(ctr, kg, o);
        w = o[0];
    }
}

/* Law 4, the strict reading of PAPER.md:404-410 (sigma_c = 0, m_c itself Gaussian): the fixed
 * period of cell c, from the spare word w3 of its initial draw (Philox ctr (0, c, 0, 1)). */
uint64_t oracle_cell_period_q32(uint64_t seed, uint64_t c) {
    const uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    uint32_t ctr[4] = {0, (uint32_t)(c & 0xffffffffu), (uint32_t)(c >> 32), 1u}, w[4];
    oracle_philox4x32_10(ctr, key, w);
    return oracle_gauss_u(w[3], w[3], (uint32_t)(c & 0xffffffffu), 10u);
}

/* Delta = max(1, (U INV) >> 32) with the tie quantisation of P3b. */
static uint64_t delta_of_u(uint64_t q, uint64_t inv_lambda, int tie_bits) {
    unsigned __int128 prod = (unsigned __int128)q * inv_lambda;
    uint64_t d = (uint64_t)(prod >> 32);
    if (d < 1) d = 1;
    if (tie_bits > 0) {
        uint64_t quantum = 1ULL << tie_bits;
        d &= ~(quantum - 1);
        if (d < quantum) d = quantum;
    }
    return d;
}

uint64_t oracle_law_q32(uint32_t w1, uint32_t w2, int law) {
    if (law == 1) return (uint64_t)w1;
    if (law == 3) return oracle_gauss_u(w1, w1, w2, 9u);   /* Gaussian period, liberal */
    if (law == 2) {
        double r = ((double)w1 + 0.5) * (1.0 / 4294967296.0);
        return (uint64_t)floor(sqrt(sqrt(sqrt(r))) * 4294967296.0);
    }
    return oracle_nlog_q32(((uint64_t)w1 << 32) | w2);
}

/* next_t = t + U / lambda; next_t > t. */
uint64_t oracle_delta_law(uint32_t w1, uint32_t w2, uint64_t inv_lambda, int tie_bits, int law) {
    return delta_of_u(oracle_law_q32(w1, w2, law), inv_lambda, tie_bits);
}

/* The increment of cell c at any arrival: law 4 uses the cell's fixed period, every other law the
 * arrival's draw (w1, w2). */
static uint64_t cell_delta(uint64_t seed, uint64_t c, uint32_t w1, uint32_t w2, uint64_t inv_lambda, int tie_bits,
                           int law) {
    if (law == 4) return delta_of_u(oracle_cell_period_q32(seed, c), inv_lambda, tie_bits);
    return oracle_delta_law(w1, w2, inv_lambda, tie_bits, law);
}

/* Eq. newt1i: next_t = t - ln(r)/lambda (the Poisson law). */
uint64_t oracle_delta(uint32_t w1, uint32_t w2, uint64_t inv_lambda, int tie_bits) {
    return oracle_delta_law(w1, w2, inv_lambda, tie_bits, 0);
}

/* ---------------------------------------------------------------- P4: flip thresholds */
/* Appendix: dE = 2(J s Sigma + H s), x = exp(-dE/T), p = x/(1+x),
 * index = (Sigma+4)/2 + 5(s+1)/2; generalised to z = 2*ndim neighbours. Metropolis
 * acceptance min(1, exp(-beta dE)) is the MRRTT rule the paper names. */
void oracle_flip_table_z(int zc, double beta, double J, double h, int rule, uint64_t* out) {
    for (int sb = 0; sb < 2; sb++) {
        int s = 2 * sb - 1;
        for (int k = 0; k <= zc; k++) {
            int sigma = 2 * k - zc;
            double dE = 2.0 * (J * (double)s * (double)sigma + h * (double)s);
            double a = beta * dE;
            double p;
            if (rule == 0) {
                if (a >= 0) { double x = exp(-a); p = x / (1.0 + x); }
                else p = 1.0 / (1.0 + exp(a));
            } else {
                p = (dE <= 0) ? 1.0 : exp(-a);
            }
            uint64_t thr = (p == 1.0) ? (1ULL << 32) : (uint64_t)floor(p * 4294967296.0);
            int idx = (sigma + zc) / 2 + (zc + 1) * (s + 1) / 2;
            out[idx] = thr;
        }
    }
}

void oracle_flip_table(int ndim, double beta, double J, double h, int rule, uint64_t* out) {
    oracle_flip_table_z(2 * ndim, beta, J, h, rule, out);
}

/* ---------------------------------------------------------------- P7 */
/* P7 event hash term (docs/PRIMITIVES.md): h = (w3 | 1) * (t ^ (l << 1) ^ s') mod 2^64, with w3
 * the fourth Philox word of the arrival's draw, t the arrival time, l the cell within the
 * subarray (0 for one-cell engines) and s' = 1 iff the new spin is +1. A checksum of our own
 * design, not arithmetic of the paper's method. */
uint64_t oracle_ev_hash(uint32_t w3, uint64_t t, uint64_t l, int new_spin) {
    return (uint64_t)(w3 | 1u) * (t ^ (l << 1) ^ (uint64_t)(new_spin > 0 ? 1 : 0));
}

/* ---------------------------------------------------------------- simulation state */
struct oracle_sim {
    int ndim, zc;
    int64_t dims[3], N;
    double lambda, beta, J, h, init_q;
    int rule, tie_bits, law;
    int q, nofs;                       /* q-th degree neighbourhood (Eq. neiq); q = 1: the 2 ndim neighbours */
    int ofs[ORACLE_MAXZ][3];           /* q > 1: the offsets of neighbors^q(c) minus c itself */
    uint64_t seed, inv_lambda, thr_init, thr[2 * (ORACLE_MAXZ + 1)];
    uint32_t key[2];
    int8_t* s;
    uint64_t* t;
    uint32_t* n;
    uint32_t* heap;
    int64_t heap_size;
    int heap_valid;
    uint64_t T_last;
    uint64_t flips, event_hash, rounds;
};

int64_t oracle_num_cells(const oracle_sim* s) { return s->N; }

/* neighbours of c with multiplicity, order -x,+x,-y,+y[,-z,+z]; periodic.
 * rule 2 (asynchronous Game of Life, P10): the 8 Moore neighbours, the same four first, then
 * (-x,-y), (+x,-y), (-x,+y), (+x,+y). */
static int neighbours(const oracle_sim* S, int64_t c, int64_t* nb) {
    int64_t nx = S->dims[0], ny = S->dims[1];
    int64_t x = c % nx, y = (c / nx) % ny, zz = (S->ndim == 3) ? c / (nx * ny) : 0;
    if (S->q > 1) {   /* neighbors^q(c) \ {c}: the offset set of q_offsets, wrapped */
        int64_t nz = S->dims[2];
        for (int j = 0; j < S->nofs; j++) {
            int64_t X = (x + S->ofs[j][0] + S->q * nx) % nx, Y = (y + S->ofs[j][1] + S->q * ny) % ny;
            int64_t Z = (zz + S->ofs[j][2] + S->q * nz) % nz;
            nb[j] = (Z * ny + Y) * nx + X;
        }
        return S->nofs;
    }
    int64_t base = c - x;
    nb[0] = base + (x + nx - 1) % nx;
    nb[1] = base + (x + 1) % nx;
    int64_t plane = zz * nx * ny;
    nb[2] = plane + ((y + ny - 1) % ny) * nx + x;
    nb[3] = plane + ((y + 1) % ny) * nx + x;
    if (S->ndim == 3) {
        int64_t nz = S->dims[2];
        nb[4] = ((zz + nz - 1) % nz) * nx * ny + y * nx + x;
        nb[5] = ((zz + 1) % nz) * nx * ny + y * nx + x;
    }
    if (S->rule == 2) {
        int64_t xm = (x + nx - 1) % nx, xp = (x + 1) % nx, ym = (y + ny - 1) % ny, yp = (y + 1) % ny;
        nb[4] = ym * nx + xm; nb[5] = ym * nx + xp; nb[6] = yp * nx + xm; nb[7] = yp * nx + xp;
    }
    return S->zc;
}

int oracle_neighbours(const oracle_sim* S, int64_t c, int64_t* nb) { return neighbours(S, c, nb); }

static void draw(const oracle_sim* S, uint32_t k, int64_t c, uint32_t tag, uint32_t w[4]) {
    uint32_t ctr[4] = {k, (uint32_t)((uint64_t)c & 0xffffffffu), (uint32_t)((uint64_t)c >> 32), tag};
    oracle_philox4x32_10(ctr, S->key, w);
}

oracle_sim* oracle_create(int ndim, const int64_t* dims, double lambda, double beta, double J,
                          double h, int rule, uint64_t seed, double init_q, int tie_bits) {
    return oracle_create_q(ndim, dims, 1, lambda, beta, J, h, rule, seed, init_q, tie_bits, 0);
}

oracle_sim* oracle_create_law(int ndim, const int64_t* dims, double lambda, double beta, double J,
                              double h, int rule, uint64_t seed, double init_q, int tie_bits, int law) {
    return oracle_create_q(ndim, dims, 1, lambda, beta, J, h, rule, seed, init_q, tie_bits, law);
}

/* Eq. neiq applied literally to offset vectors: neighbors^1 = the cell and
 * its 2 ndim first-degree neighbours; neighbors^q = neighbors(neighbors^(q-1)), the union of the
 * first-degree neighbourhoods of its members. Returns the members other than the cell itself
 * (their number is |neighbors^q(c)| - 1), or -1 if there are more than `cap`. On the torus the
 * set is the same around every cell (translation), so it is computed once around the origin. */
int oracle_q_offsets(int ndim, int q, int (*out)[3], int cap) {
    int set[2 * ORACLE_MAXZ + 2][3], n = 1, nxt[2 * ORACLE_MAXZ + 2][3];
    set[0][0] = set[0][1] = set[0][2] = 0;
    for (int k = 1; k <= q; k++) {
        int m = 0;
        for (int i = 0; i < n; i++) {
            for (int d = -1; d < 2 * ndim; d++) {   /* d = -1: the member itself (c is in neighbors(c)) */
                int v[3] = {set[i][0], set[i][1], set[i][2]};
                if (d >= 0) v[d / 2] += (d % 2) ? 1 : -1;
                int dup = 0;
                for (int j = 0; j < m && !dup; j++)
                    dup = nxt[j][0] == v[0] && nxt[j][1] == v[1] && nxt[j][2] == v[2];
                if (dup) continue;
                if (m == 2 * ORACLE_MAXZ + 2) return -1;
                nxt[m][0] = v[0]; nxt[m][1] = v[1]; nxt[m][2] = v[2]; m++;
            }
        }
        memcpy(set, nxt, sizeof(int) * 3 * (size_t)m);
        n = m;
    }
    int r = 0;
    for (int i = 0; i < n; i++) {
        if (!set[i][0] && !set[i][1] && !set[i][2]) continue;
        if (r == cap) return -1;
        out[r][0] = set[i][0]; out[r][1] = set[i][1]; out[r][2] = set[i][2]; r++;
    }
    return r;
}

/* q >= 2: the Ising model on neighbors^q (docs/PRIMITIVES.md P12): Sigma sums
 * the spins of neighbors^q(c) \ {c}, the P4 table has z = |neighbors^q| - 1, a cell fires when its
 * (t, c) is below every member's. Every side must be >= 2q + 1 so the members are distinct cells. */
oracle_sim* oracle_create_q(int ndim, const int64_t* dims, int q, double lambda, double beta, double J,
                            double h, int rule, uint64_t seed, double init_q, int tie_bits, int law) {
    if (ndim != 2 && ndim != 3) return NULL;
    if (q < 1 || q > 4) return NULL;
    if (q > 1) {
        if (rule == 2) return NULL;
        for (int a = 0; a < ndim; a++) if (dims[a] < 2 * q + 1) return NULL;
    }
    if (law < 0 || law > 4) return NULL;
    if (!(lambda > 0) || !isfinite(lambda) || !(beta >= 0) || !isfinite(beta)) return NULL;
    if (rule != 0 && rule != 1 && !(rule == 2 && ndim == 2)) return NULL;
    if (!(init_q >= 0 && init_q <= 1)) return NULL;
    if (tie_bits < 0 || tie_bits > 40) return NULL;
    int64_t N = 1;
    for (int a = 0; a < ndim; a++) { if (dims[a] < 2) return NULL; N *= dims[a]; }
    if (N >= (1LL << 32)) return NULL;
    oracle_sim* S = (oracle_sim*)calloc(1, sizeof(oracle_sim));
    S->ndim = ndim; S->zc = rule == 2 ? 8 : 2 * ndim; S->N = N;
    S->q = q;
    if (q > 1) {
        S->nofs = oracle_q_offsets(ndim, q, S->ofs, ORACLE_MAXZ);
        if (S->nofs < 0) { free(S); return NULL; }
        S->zc = S->nofs;
    }
    for (int a = 0; a < 3; a++) S->dims[a] = a < ndim ? dims[a] : 1;
    S->lambda = lambda; S->beta = beta; S->J = J; S->h = h; S->rule = rule;
    S->seed = seed; S->init_q = init_q; S->tie_bits = tie_bits; S->law = law;
    S->inv_lambda = oracle_inv_lambda(lambda);
    S->thr_init = (uint64_t)floor(init_q * 4294967296.0);
    oracle_flip_table_z(S->zc, beta, J, h, rule, S->thr);
    S->key[0] = (uint32_t)(seed & 0xffffffffu);
    S->key[1] = (uint32_t)(seed >> 32);
    S->s = (int8_t*)malloc((size_t)N);
    S->t = (uint64_t*)malloc((size_t)N * 8);
    S->n = (uint32_t*)malloc((size_t)N * 4);
    S->heap = NULL;
    if (!S->s || !S->t || !S->n) { oracle_destroy(S); return NULL; }
    /* P5: one initial draw per cell; local clocks start at 0. */
    for (int64_t c = 0; c < N; c++) {
        uint32_t w[4];
        draw(S, 0, c, 1u, w);
        S->s[c] = ((uint64_t)w[0] < S->thr_init) ? -1 : 1;
        S->t[c] = cell_delta(seed, (uint64_t)c, w[1], w[2], S->inv_lambda, tie_bits, law);
        S->n[c] = 0;
    }
    return S;
}

void oracle_destroy(oracle_sim* S) {
    if (!S) return;
    free(S->s); free(S->t); free(S->n); free(S->heap);
    free(S);
}

/* One arrival of cell c (fig:a1c1pe steps 3-4; Appendix):
 * Sigma from the neighbours' current spins (the "just before" states),
 * flip iff w0 < thr[idx], then t += Delta, n += 1. new_s / new_t are returned so the
 * synchronous variant can commit them later. */
static void arrival(oracle_sim* S, int64_t c, int8_t* new_s, uint64_t* new_t) {
    int64_t nb[ORACLE_MAXZ];
    int z = neighbours(S, c, nb);
    int sigma = 0;
    for (int j = 0; j < z; j++) sigma += S->s[nb[j]];
    int sc = S->s[c];
    uint32_t k = S->n[c];
    uint32_t w[4];
    draw(S, k, c, 0u, w);
    int ns = sc;
    if (S->rule == 2) {   /* P10: Conway's rule on the Moore neighbourhood, deterministic */
        int live = (sigma + z) / 2;
        ns = (live == 3 || (sc > 0 && live == 2)) ? 1 : -1;
        if (ns != sc) S->flips++;
    } else {
        int idx = (sigma + z) / 2 + (z + 1) * (sc + 1) / 2;
        if ((uint64_t)w[0] < S->thr[idx]) { ns = -sc; S->flips++; }
    }
    uint64_t tev = S->t[c];
    S->event_hash += oracle_ev_hash(w[3], tev, 0, ns);
    *new_s = (int8_t)ns;
    *new_t = tev + cell_delta(S->seed, (uint64_t)c, w[1], w[2], S->inv_lambda, S->tie_bits, S->law);
}

/* lexicographic (t, c) order (P6). */
static int lex_less(const oracle_sim* S, int64_t a, int64_t b) {
    return S->t[a] < S->t[b] || (S->t[a] == S->t[b] && a < b);
}

static void sift_down(oracle_sim* S, int64_t i) {
    int64_t n = S->heap_size;
    uint32_t* H = S->heap;
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < n && lex_less(S, H[l], H[m])) m = l;
        if (r < n && lex_less(S, H[r], H[m])) m = r;
        if (m == i) return;
        uint32_t tmp = H[i]; H[i] = H[m]; H[m] = tmp;
        i = m;
    }
}

static void build_heap(oracle_sim* S) {
    if (!S->heap) S->heap = (uint32_t*)malloc((size_t)S->N * 4);
    for (int64_t c = 0; c < S->N; c++) S->heap[c] = (uint32_t)c;
    S->heap_size = S->N;
    for (int64_t i = S->N / 2 - 1; i >= 0; i--) sift_down(S, i);
    S->heap_valid = 1;
}

/* (A) The oracle: global priority queue on (t(c), c); pop while t < T. */
int oracle_run_until_q32(oracle_sim* S, uint64_t T) {
    if (T < S->T_last) return -1;
    S->T_last = T;
    if (!S->heap_valid) build_heap(S);
    while (S->heap_size > 0) {
        int64_t c = S->heap[0];
        if (S->t[c] >= T) break;
        int8_t ns; uint64_t nt;
        arrival(S, c, &ns, &nt);
        S->s[c] = ns; S->t[c] = nt; S->n[c] += 1;
        sift_down(S, 0);   /* the popped key only grew: re-insert by sifting the root */
    }
    return 0;
}

/* (D) The same global priority queue on (t, c) as (A), organised as a calendar queue (SURVEY
 * 8(c) step 2: "a calendar/bucket queue that is exact on (t, c)"): pending arrivals are kept in
 * buckets of width 2^BSH Q32 units by t >> BSH, on a ring longer than any increment; the bucket in
 * progress is a binary heap on (t, c), later buckets are unsorted lists. Every arrival of an
 * earlier bucket precedes every arrival of a later one, and within the bucket the heap pops in
 * (t, c) order, so the events are processed in exactly the order of (A) — the same trajectory,
 * bit for bit (tests/test_oracle_sim.py pins (D) == (A)) — with memory traffic local to one
 * bucket instead of a heap over the whole lattice. Used for the long full-lattice golden runs. */
typedef struct { uint64_t t; uint32_t c; } cq_ev;
typedef struct { cq_ev* v; int64_t n, cap; } cq_list;

static int cq_less(cq_ev a, cq_ev b) { return a.t < b.t || (a.t == b.t && a.c < b.c); }
static int cq_push(cq_list* L, cq_ev e) {
    if (L->n == L->cap) {
        int64_t nc = L->cap ? 2 * L->cap : 64;
        cq_ev* nv = (cq_ev*)realloc(L->v, (size_t)nc * sizeof(cq_ev));
        if (!nv) return -1;
        L->v = nv; L->cap = nc;
    }
    L->v[L->n++] = e;
    return 0;
}
static void cq_sift_down(cq_ev* H, int64_t n, int64_t i) {
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < n && cq_less(H[l], H[m])) m = l;
        if (r < n && cq_less(H[r], H[m])) m = r;
        if (m == i) return;
        cq_ev tmp = H[i]; H[i] = H[m]; H[m] = tmp;
        i = m;
    }
}
static void cq_sift_up(cq_ev* H, int64_t i) {
    while (i > 0) {
        int64_t p = (i - 1) / 2;
        if (!cq_less(H[i], H[p])) return;
        cq_ev tmp = H[i]; H[i] = H[p]; H[p] = tmp;
        i = p;
    }
}

int oracle_run_until_calendar(oracle_sim* S, uint64_t T) {
    if (T < S->T_last) return -1;
    S->T_last = T;
    S->heap_valid = 0;   /* (A) rebuilds its heap from the state next time */
    const int BSH = 26;  /* bucket width 2^26 Q32 units = 1/64 of a time unit */
    /* ring length: more buckets than the largest increment spans (law 0: NLOG-2 <= 190530846196
     * at lambda = 1; every law's increment is below 64 ln 2 / lambda time units) */
    uint64_t maxd = ((uint64_t)190530846196ULL >> 16) * (S->inv_lambda >> 16) + (1ULL << 33);
    if (S->tie_bits) maxd += 1ULL << S->tie_bits;
    int64_t R = 1;
    while ((uint64_t)R <= (maxd >> BSH) + 2) R <<= 1;
    cq_list* B = (cq_list*)calloc((size_t)R, sizeof(cq_list));
    if (!B) return -2;
    uint64_t tmin = ~0ULL;
    for (int64_t c = 0; c < S->N; c++) {
        if (S->t[c] >= T) continue;
        cq_ev e = {S->t[c], (uint32_t)c};
        if (cq_push(&B[(S->t[c] >> BSH) & (uint64_t)(R - 1)], e)) return -2;
        if (S->t[c] < tmin) tmin = S->t[c];
    }
    int rc = 0;
    if (tmin != ~0ULL) {
        uint64_t b = tmin >> BSH;          /* absolute index of the bucket in progress */
        const uint64_t bend = (T - 1) >> BSH;
        for (; b <= bend; b++) {
            cq_list* L = &B[b & (uint64_t)(R - 1)];
            cq_ev* H = L->v;
            for (int64_t i = L->n / 2 - 1; i >= 0; i--) cq_sift_down(H, L->n, i);
            while (L->n > 0) {
                H = L->v;
                const int64_t c = H[0].c;
                H[0] = H[--L->n];
                cq_sift_down(H, L->n, 0);
                int8_t ns; uint64_t nt;
                arrival(S, c, &ns, &nt);
                S->s[c] = ns; S->t[c] = nt; S->n[c] += 1;
                if (nt >= T) continue;
                cq_ev e = {nt, (uint32_t)c};
                const uint64_t nb = nt >> BSH;
                if (nb == b) {   /* the same bucket: into its heap */
                    if (cq_push(L, e)) { rc = -2; break; }
                    cq_sift_up(L->v, L->n - 1);
                } else if (cq_push(&B[nb & (uint64_t)(R - 1)], e)) { rc = -2; break; }
            }
            if (rc) break;
            free(L->v);   /* drained: release it, or every ring slot keeps its peak capacity */
            L->v = NULL;
            L->cap = 0;
        }
    }
    for (int64_t i = 0; i < R; i++) free(B[i].v);
    free(B);
    return rc;
}

/* eligibility: fig:a1c1pe step 2 with the (t, c) tie-break (P6).
 * naive_leq = 1 is a NEGATIVE CONTROL only: the bare "t(c) <= min t(c')" test of
 * fig:s1c1pe without a tie-break, which lets tied neighbours fire in the same round. */
static int eligible_rule(const oracle_sim* S, int64_t c, uint64_t T, int naive_leq) {
    if (S->t[c] >= T) return 0;
    int64_t nb[ORACLE_MAXZ];
    int z = neighbours(S, c, nb);
    for (int j = 0; j < z; j++) {
        if (naive_leq ? !(S->t[c] <= S->t[nb[j]]) : !lex_less(S, c, nb[j])) return 0;
    }
    return 1;
}
static int eligible(const oracle_sim* S, int64_t c, uint64_t T) { return eligible_rule(S, c, T, 0); }

/* (B) uniformly random eligible local minimum, any order. */
int oracle_run_until_random_order(oracle_sim* S, uint64_t T, uint64_t choice_seed) {
    if (T < S->T_last) return -1;
    S->T_last = T;
    S->heap_valid = 0;
    int64_t N = S->N;
    int64_t* pos = (int64_t*)malloc((size_t)N * 8);
    int64_t* set = (int64_t*)malloc((size_t)N * 8);
    int64_t size = 0;
    for (int64_t c = 0; c < N; c++) {
        pos[c] = -1;
        if (eligible(S, c, T)) { pos[c] = size; set[size++] = c; }
    }
    uint64_t rs = choice_seed * 2654435761ULL + 0x9E3779B97F4A7C15ULL;
    if (!rs) rs = 1;
    while (size > 0) {
        rs ^= rs >> 12; rs ^= rs << 25; rs ^= rs >> 27;          /* xorshift64* */
        uint64_t r = rs * 2685821657736338717ULL;
        int64_t c = set[(int64_t)(r % (uint64_t)size)];
        int8_t ns; uint64_t nt;
        arrival(S, c, &ns, &nt);
        S->s[c] = ns; S->t[c] = nt; S->n[c] += 1;
        int64_t touch[ORACLE_MAXZ + 1];
        touch[0] = c;
        int z = neighbours(S, c, touch + 1);
        for (int j = 0; j <= z; j++) {
            int64_t d = touch[j];
            int e = eligible(S, d, T);
            if (e && pos[d] < 0) { pos[d] = size; set[size++] = d; }
            else if (!e && pos[d] >= 0) {
                int64_t p = pos[d], last = set[--size];
                set[p] = last; pos[last] = p; pos[d] = -1;
            }
        }
    }
    free(pos); free(set);
    return 0;
}

/* (C) fig:s1c1pe: round = test all (step 2), compute new_s/new_t
 * privately (steps 3-4), barrier, commit (steps 6-7). */
static int64_t run_sync(oracle_sim* S, uint64_t T, uint64_t* fired_per_round,
                        int64_t max_rounds, int naive_leq);
int64_t oracle_run_until_sync(oracle_sim* S, uint64_t T, uint64_t* fired_per_round,
                              int64_t max_rounds) {
    return run_sync(S, T, fired_per_round, max_rounds, 0);
}
int64_t oracle_run_until_sync_naive_leq(oracle_sim* S, uint64_t T) {
    return run_sync(S, T, NULL, 0, 1);
}
static int64_t run_sync(oracle_sim* S, uint64_t T, uint64_t* fired_per_round,
                        int64_t max_rounds, int naive_leq) {
    if (T < S->T_last) return -1;
    S->T_last = T;
    S->heap_valid = 0;
    int64_t N = S->N, rounds = 0;
    int64_t* list = (int64_t*)malloc((size_t)N * 8);
    int8_t* ns = (int8_t*)malloc((size_t)N);
    uint64_t* nt = (uint64_t*)malloc((size_t)N * 8);
    for (;;) {
        int64_t m = 0;
        for (int64_t c = 0; c < N; c++) if (eligible_rule(S, c, T, naive_leq)) list[m++] = c;
        if (m == 0) break;
        for (int64_t j = 0; j < m; j++) arrival(S, list[j], &ns[j], &nt[j]);
        for (int64_t j = 0; j < m; j++) {
            int64_t c = list[j];
            S->s[c] = ns[j]; S->t[c] = nt[j]; S->n[c] += 1;
        }
        if (fired_per_round && rounds < max_rounds) fired_per_round[rounds] = (uint64_t)m;
        rounds++;
    }
    S->rounds += (uint64_t)rounds;
    free(list); free(ns); free(nt);
    return rounds;
}

void oracle_get_spins(const oracle_sim* S, int8_t* out) { memcpy(out, S->s, (size_t)S->N); }
void oracle_get_times(const oracle_sim* S, uint64_t* out) { memcpy(out, S->t, (size_t)S->N * 8); }
void oracle_get_counters(const oracle_sim* S, uint32_t* out) { memcpy(out, S->n, (size_t)S->N * 4); }

/* Energy bookkeeping, Appendix comment "Energy = -J sum spin spin' - H sum spin"
 * (PAPER.md:1680): B counts each bond once along +e_a, periodic; with neighbors^q (q > 1) each
 * pair of cells within it once. */
void oracle_get_stats(const oracle_sim* S, oracle_stats* o) {
    memset(o, 0, sizeof(*o));
    int64_t nb[ORACLE_MAXZ];
    uint64_t tmin = ~0ULL, tmax = 0, arr = 0;
    int64_t B = 0, B2 = 0, M = 0;
    for (int64_t c = 0; c < S->N; c++) {
        int z = neighbours(S, c, nb);
        int sc = S->s[c];
        if (S->q > 1) {   /* each pair {c, c'} of neighbors^q appears twice in the double sum */
            int all = 0;
            for (int j = 0; j < z; j++) all += S->s[nb[j]];
            B2 += sc * all;
        } else {
            int plus = S->s[nb[1]] + S->s[nb[3]] + (S->ndim == 3 ? S->s[nb[5]] : 0);
            B += sc * plus;
        }
        M += sc;
        arr += S->n[c];
        if (S->t[c] < tmin) tmin = S->t[c];
        if (S->t[c] > tmax) tmax = S->t[c];
    }
    if (S->q > 1) B = B2 / 2;
    o->arrivals = arr; o->flips = S->flips; o->event_hash = S->event_hash;
    o->bond_sum = B; o->magnetisation = M; o->t_min = tmin; o->t_max = tmax;
    o->rounds = S->rounds;
}

/* ---------------------------------------------------------------- Boltzmann helpers */
static uint64_t state_code(const oracle_sim* S) {
    uint64_t code = 0;
    for (int64_t c = 0; c < S->N; c++) if (S->s[c] > 0) code |= 1ULL << c;
    return code;
}

int oracle_replica_hist(int ndim, const int64_t* dims, double beta, double J, double h,
                        int rule, uint64_t seed0, int64_t n_rep, uint64_t T, uint64_t* hist) {
    for (int64_t r = 0; r < n_rep; r++) {
        oracle_sim* S = oracle_create(ndim, dims, 1.0, beta, J, h, rule, seed0 + (uint64_t)r, 0.5, 0);
        if (!S || S->N > 20) { oracle_destroy(S); return -1; }
        oracle_run_until_q32(S, T);
        hist[state_code(S)] += 1;
        oracle_destroy(S);
    }
    return 0;
}

int oracle_time_weighted_hist(int ndim, const int64_t* dims, double beta, double J, double h,
                              int rule, uint64_t seed, uint64_t T0, uint64_t T1, double* weight) {
    oracle_sim* S = oracle_create(ndim, dims, 1.0, beta, J, h, rule, seed, 0.5, 0);
    if (!S || S->N > 20) { oracle_destroy(S); return -1; }
    oracle_run_until_q32(S, T0);
    uint64_t code = state_code(S), tprev = T0;
    S->T_last = T1;
    while (S->heap_size > 0) {
        int64_t c = S->heap[0];
        if (S->t[c] >= T1) break;
        uint64_t tev = S->t[c];
        weight[code] += (double)(tev - tprev) * (1.0 / 4294967296.0);
        tprev = tev;
        int8_t ns; uint64_t nt;
        arrival(S, c, &ns, &nt);
        S->s[c] = ns; S->t[c] = nt; S->n[c] += 1;
        sift_down(S, 0);
        if (ns > 0) code |= 1ULL << c; else code &= ~(1ULL << c);
    }
    weight[code] += (double)(T1 - tprev) * (1.0 / 4294967296.0);
    oracle_destroy(S);
    return 0;
}

/* ---------------------------------------------------------------- per-cell closed forms */
void oracle_nlog_batch(int64_t n, const uint64_t* X, uint64_t* q) {
    for (int64_t i = 0; i < n; i++) q[i] = oracle_nlog_q32(X[i]);
}

/* Arrival times are state-independent for Ising: cell c's pending
 * time and counter after run_until(T) follow from its own stream alone. */
void oracle_cell_time_counter(uint64_t seed, uint64_t c, uint64_t T_q32, uint64_t inv_lambda,
                              int tie_bits, uint64_t* t_out, uint32_t* n_out) {
    oracle_cell_time_counter_law(seed, c, T_q32, inv_lambda, tie_bits, 0, t_out, n_out);
}

void oracle_cell_time_counter_law(uint64_t seed, uint64_t c, uint64_t T_q32, uint64_t inv_lambda,
                                  int tie_bits, int law, uint64_t* t_out, uint32_t* n_out) {
    uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    uint32_t ctr[4] = {0, (uint32_t)(c & 0xffffffffu), (uint32_t)(c >> 32), 1u};
    uint32_t w[4];
    oracle_philox4x32_10(ctr, key, w);
    uint64_t t = cell_delta(seed, c, w[1], w[2], inv_lambda, tie_bits, law);
    uint32_t k = 0;
    while (t < T_q32) {
        uint32_t ce[4] = {k, (uint32_t)(c & 0xffffffffu), (uint32_t)(c >> 32), 0u};
        oracle_philox4x32_10(ce, key, w);
        t += cell_delta(seed, c, w[1], w[2], inv_lambda, tie_bits, law);
        k++;
    }
    *t_out = t;
    *n_out = k;
}

/* ---------------------------------------------------------------- window (light-cone) oracle
 * Exact (s, t, n) of one cell of a lattice too large to simulate whole. A box of radius
 * `radius` around the cell is simulated in (t, c) order with the cells' true global ids and
 * streams; times and counters are exact everywhere (state-independent).
 * A cell's spin is exact unless information from outside the box can have reached it: a
 * cell becomes "unknown" when it processes an arrival whose flip decision depends on an
 * unknown neighbour spin (a neighbour outside the box or itself unknown). With refine = 1 a
 * decision that comes out the same for every possible value of the unknown spins stays
 * exact (e.g. a rejection at low temperature). Causality (fig:amcgen):
 * known spins are the true spins. *exact_out = 0 if the target ended unknown (enlarge the box). */
typedef struct { uint64_t t; uint64_t gc; int64_t lc; } wev;

static int wev_less(const wev* a, const wev* b) { return a->t < b->t || (a->t == b->t && a->gc < b->gc); }

int oracle_window_cell(int ndim, const int64_t* dims, double lambda, double beta, double J, double h, int rule,
                       uint64_t seed, double init_q, int tie_bits, uint64_t T, const int64_t* center,
                       int64_t radius, int refine, int8_t* s_out, uint64_t* t_out, uint32_t* n_out,
                       int* exact_out) {
    return oracle_window_cell_law(ndim, dims, lambda, beta, J, h, rule, seed, init_q, tie_bits, T, center, radius,
                                  refine, s_out, t_out, n_out, exact_out, 0);
}

int oracle_window_cell_law(int ndim, const int64_t* dims, double lambda, double beta, double J, double h, int rule,
                       uint64_t seed, double init_q, int tie_bits, uint64_t T, const int64_t* center,
                       int64_t radius, int refine, int8_t* s_out, uint64_t* t_out, uint32_t* n_out,
                       int* exact_out, int law) {
    if (rule == 2) return -1;   /* the window oracle covers the Ising rules only */
    int64_t D[3] = {1, 1, 1}, W[3] = {1, 1, 1}, lo[3] = {0, 0, 0};
    int fullax[3] = {1, 1, 1};
    int64_t NW = 1;
    for (int a = 0; a < ndim; a++) {
        D[a] = dims[a];
        if (2 * radius + 1 >= D[a]) { W[a] = D[a]; lo[a] = 0; fullax[a] = 1; }
        else { W[a] = 2 * radius + 1; lo[a] = center[a] - radius; fullax[a] = 0; }
        NW *= W[a];
    }
    int zc = 2 * ndim;
    uint64_t thr[14];
    oracle_flip_table(ndim, beta, J, h, rule, thr);
    uint64_t inv = oracle_inv_lambda(lambda);
    uint64_t thr_init = (uint64_t)floor(init_q * 4294967296.0);
    uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    int8_t* s = (int8_t*)malloc((size_t)NW);
    uint8_t* unk = (uint8_t*)calloc((size_t)NW, 1);
    uint64_t* t = (uint64_t*)malloc((size_t)NW * 8);
    uint32_t* n = (uint32_t*)calloc((size_t)NW, 4);
    uint64_t* gid = (uint64_t*)malloc((size_t)NW * 8);
    int64_t* nb = (int64_t*)malloc((size_t)NW * 6 * 8);    /* -1: outside the box */
    wev* heap = (wev*)malloc((size_t)NW * sizeof(wev));
    if (!s || !unk || !t || !n || !gid || !nb || !heap) return -1;
    for (int64_t l = 0; l < NW; l++) {
        int64_t lx = l % W[0], ly = (l / W[0]) % W[1], lz = l / (W[0] * W[1]);
        int64_t L[3] = {lx, ly, lz}, G[3];
        for (int a = 0; a < 3; a++) G[a] = (((lo[a] + L[a]) % D[a]) + D[a]) % D[a];
        gid[l] = (uint64_t)((G[2] * D[1] + G[1]) * D[0] + G[0]);
        for (int a = 0; a < ndim; a++) {
            for (int dir = 0; dir < 2; dir++) {
                int64_t M[3] = {L[0], L[1], L[2]};
                M[a] += dir ? 1 : -1;
                int64_t r;
                if (fullax[a]) { M[a] = (M[a] + W[a]) % W[a]; r = (M[2] * W[1] + M[1]) * W[0] + M[0]; }
                else if (M[a] < 0 || M[a] >= W[a]) r = -1;
                else r = (M[2] * W[1] + M[1]) * W[0] + M[0];
                nb[l * 6 + 2 * a + dir] = r;
            }
        }
        uint32_t ctr[4] = {0, (uint32_t)(gid[l] & 0xffffffffu), (uint32_t)(gid[l] >> 32), 1u}, w[4];
        oracle_philox4x32_10(ctr, key, w);
        s[l] = ((uint64_t)w[0] < thr_init) ? -1 : 1;
        t[l] = cell_delta(seed, gid[l], w[1], w[2], inv, tie_bits, law);
    }
    /* binary heap of (t, global id, local id) */
    int64_t hn = 0;
    for (int64_t l = 0; l < NW; l++) {
        wev e = {t[l], gid[l], l};
        int64_t i = hn++;
        heap[i] = e;
        while (i > 0) {
            int64_t p = (i - 1) / 2;
            if (!wev_less(&heap[i], &heap[p])) break;
            wev tmp = heap[i]; heap[i] = heap[p]; heap[p] = tmp; i = p;
        }
    }
    while (hn > 0 && heap[0].t < T) {
        int64_t c = heap[0].lc;
        int known = 0, u = 0;
        for (int j = 0; j < zc; j++) {
            int64_t m = nb[c * 6 + j];
            if (m < 0 || unk[m]) u++; else known += s[m];
        }
        uint32_t ctr[4] = {n[c], (uint32_t)(gid[c] & 0xffffffffu), (uint32_t)(gid[c] >> 32), 0u}, w[4];
        oracle_philox4x32_10(ctr, key, w);
        if (!unk[c]) {
            int sc = s[c];
            if (u == 0) {
                int idx = (known + zc) / 2 + (zc + 1) * (sc + 1) / 2;
                if ((uint64_t)w[0] < thr[idx]) s[c] = (int8_t)-sc;
            } else if (refine) {
                int f0 = -1, same = 1;
                for (int k = 0; k <= u; k++) {
                    int sigma = known + 2 * k - u;
                    int idx = (sigma + zc) / 2 + (zc + 1) * (sc + 1) / 2;
                    int f = (uint64_t)w[0] < thr[idx];
                    if (f0 < 0) f0 = f; else if (f != f0) same = 0;
                }
                if (same) { if (f0) s[c] = (int8_t)-sc; }
                else unk[c] = 1;
            } else {
                unk[c] = 1;
            }
        }
        t[c] += cell_delta(seed, gid[c], w[1], w[2], inv, tie_bits, law);
        n[c] += 1;
        heap[0].t = t[c];
        int64_t i = 0;
        for (;;) {
            int64_t l = 2 * i + 1, r = l + 1, m = i;
            if (l < hn && wev_less(&heap[l], &heap[m])) m = l;
            if (r < hn && wev_less(&heap[r], &heap[m])) m = r;
            if (m == i) break;
            wev tmp = heap[i]; heap[i] = heap[m]; heap[m] = tmp; i = m;
        }
    }
    int64_t L[3] = {0, 0, 0};
    for (int a = 0; a < ndim; a++) L[a] = fullax[a] ? center[a] : radius;
    int64_t tc = (L[2] * W[1] + L[1]) * W[0] + L[0];
    *s_out = s[tc]; *t_out = t[tc]; *n_out = n[tc]; *exact_out = !unk[tc];
    free(s); free(unk); free(t); free(n); free(gid); free(nb); free(heap);
    return 0;
}

/* ---------------------------------------------------------------- time-only efficiency model
 * for an Ising model next_t is independent of the states, so whether a
 * cell passes the test of fig:s1c1pe step 2 depends on the local times only. One iteration:
 * every cell whose (t, c) is below every neighbour's (t', c') (P6 order) increments its time;
 * all tests see the times of the previous iteration (synchronous). fired_per_round[r] = N0
 * of iteration r; the efficiency of the iteration is N0/N.
 * Draws: initial t(c) = Delta of Philox ctr (0, c, 0, TAG_INIT = 1) (P5); the increment of
 * iteration r uses ctr (r, c_lo, c_hi, TAG_EFF = 2) (a cell fires at most once per iteration).
 * ndim 1 (n-circle), 2 (torus), 3 (periodic cube); laws as P3L. Plain loops, test
 * infrastructure only. Returns 0, or -1 on bad arguments. */
int oracle_efficiency_run(int ndim, const int64_t* dims, int law, double lambda, uint64_t seed, int64_t rounds,
                          uint64_t* fired_per_round, uint64_t* t_out) {
    return oracle_efficiency_run_q(ndim, dims, law, lambda, seed, rounds, 1, fired_per_round, t_out);
}

/* ---------------------------------------------------------------- fig:perfbl model (P11)
 * The simplified many-cells-per-PE model of PAPER.md:1491-1546 (Eq. hC), in the reading where a
 * PE that selected a cell keeps it while blocked (fig:amcpoi Steps 2-3), with
 * the lag bound of PAPER.md:1573-1605. A px x py torus of PEs; PE C (= y px + x) holds h(C) (Q32)
 * and n(C). Its event n uses the draw (w0..w3) = Philox ctr (n, C, 0, 7): category 0 (the cell
 * has no outside neighbour, probability (m-2)^2/m^2) iff w0 < E1, category 1 (an edge cell,
 * 4(m-2)/m^2) iff E1 <= w0 < E2, else category 2 (a corner, 4/m^2), with
 * E1 = floor((m-2)^2 2^32 / m^2), E2 = floor((m^2-4) 2^32 / m^2); neighbour directions
 * a = w1 >> 30 and b = (a + 1 + (((w1 & 0xffff) * 3) >> 16)) & 3 (0 -x, 1 +x, 2 -y, 3 +y); the
 * increment max(1, NLOG-2((w2 << 32) | w3)) (Exp(1) in Q32: h = lambda T, time measured in
 * units of a cell's mean inter-arrival time, the unit of the lag in fig:perfbl). h0(C) = the
 * increment of the draw ctr (0, C, 0, 8). A round reads one snapshot hs of every h: hmin = min
 * hs; PE C advances (h = hs(C) + increment, n += 1) iff (lag = 0 or hs(C) < hmin + lag) and every
 * neighbour its category checks (a; a and b) has hs(C') >= hs(C) (Eq. hC conditions (i)-(iii));
 * otherwise it keeps its event. ups[r] = PEs that advanced in round r: the efficiency is their
 * mean over PEs (Eq. effi). Plain loops; test infrastructure only. 0, or -1 on bad arguments. */
int oracle_perfbl_run(int64_t px, int64_t py, int m, uint64_t lag_q32, uint64_t seed, int64_t rounds, uint64_t* ups,
                      uint64_t* h_out, uint32_t* n_out) {
    if (px < 1 || py < 1 || m < 2 || m > 65535 || rounds < 0) return -1;
    const int64_t N = px * py;
    const uint64_t mm = (uint64_t)m * (uint64_t)m;
    const uint64_t E1 = ((uint64_t)(m - 2) * (uint64_t)(m - 2) << 32) / mm, E2 = ((mm - 4) << 32) / mm;
    const uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    uint64_t* h = (uint64_t*)malloc((size_t)N * 8);
    uint64_t* hs = (uint64_t*)malloc((size_t)N * 8);
    uint32_t* n = (uint32_t*)calloc((size_t)N, 4);
    if (!h || !hs || !n) { free(h); free(hs); free(n); return -1; }
    for (int64_t C = 0; C < N; C++) {
        uint32_t ctr[4] = {0, (uint32_t)C, (uint32_t)((uint64_t)C >> 32), 8u}, w[4];
        oracle_philox4x32_10(ctr, key, w);
        uint64_t d = oracle_nlog_q32(((uint64_t)w[2] << 32) | w[3]);
        h[C] = d < 1 ? 1 : d;
    }
    for (int64_t r = 0; r < rounds; r++) {
        memcpy(hs, h, (size_t)N * 8);
        uint64_t hmin = hs[0], cnt = 0;
        for (int64_t C = 1; C < N; C++) hmin = hs[C] < hmin ? hs[C] : hmin;
        for (int64_t C = 0; C < N; C++) {
            if (lag_q32 && hs[C] - hmin >= lag_q32) continue;          /* beyond the lag window */
            uint32_t ctr[4] = {n[C], (uint32_t)C, (uint32_t)((uint64_t)C >> 32), 7u}, w[4];
            oracle_philox4x32_10(ctr, key, w);
            const int cat = (uint64_t)w[0] < E1 ? 0 : ((uint64_t)w[0] < E2 ? 1 : 2);
            const int a = (int)(w[1] >> 30), b = (a + 1 + (int)(((w[1] & 0xffffu) * 3u) >> 16)) & 3;
            const int64_t x = C % px, y = C / px;
            int64_t nb[4];
            nb[0] = y * px + (x + px - 1) % px;
            nb[1] = y * px + (x + 1) % px;
            nb[2] = ((y + py - 1) % py) * px + x;
            nb[3] = ((y + 1) % py) * px + x;
            int go = 1;
            if (cat >= 1 && hs[nb[a]] < hs[C]) go = 0;
            if (cat == 2 && hs[nb[b]] < hs[C]) go = 0;
            if (!go) continue;
            uint64_t d = oracle_nlog_q32(((uint64_t)w[2] << 32) | w[3]);
            h[C] = hs[C] + (d < 1 ? 1 : d);
            n[C] += 1;
            cnt++;
        }
        if (ups) ups[r] = cnt;
    }
    if (h_out) memcpy(h_out, h, (size_t)N * 8);
    if (n_out) memcpy(n_out, n, (size_t)N * 4);
    free(h); free(hs); free(n);
    return 0;
}

/* q-th degree neighbourhood (Eq. neiq): neighbors^q(c) =
 * neighbors(neighbors^(q-1)(c)), i.e. every cell within Manhattan distance q; a cell passes the
 * test when its (t, c) is below all of them. q = 1 is the model above. */
int oracle_efficiency_run_q(int ndim, const int64_t* dims, int law, double lambda, uint64_t seed, int64_t rounds,
                            int q, uint64_t* fired_per_round, uint64_t* t_out) {
    if (q < 1 || q > 8) return -1;
    if (ndim < 1 || ndim > 3 || law < 0 || law > 3 || !(lambda > 0) || rounds < 0) return -1;   /* law 4: n/a */
    int64_t d[3] = {1, 1, 1}, N = 1;
    for (int a = 0; a < ndim; a++) { if (dims[a] < 2) return -1; d[a] = dims[a]; N *= dims[a]; }
    uint64_t inv = oracle_inv_lambda(lambda);
    uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    uint64_t* t = (uint64_t*)malloc((size_t)N * 8);
    unsigned char* fire = (unsigned char*)malloc((size_t)N);
    if (!t || !fire) { free(t); free(fire); return -1; }
    for (int64_t c = 0; c < N; c++) {
        uint32_t ctr[4] = {0, (uint32_t)((uint64_t)c & 0xffffffffu), (uint32_t)((uint64_t)c >> 32), 1u}, w[4];
        oracle_philox4x32_10(ctr, key, w);
        t[c] = oracle_delta_law(w[1], w[2], inv, 0, law);
    }
    for (int64_t r = 0; r < rounds; r++) {
        uint64_t n0 = 0;
        for (int64_t c = 0; c < N; c++) {          /* test: all against the same times */
            int64_t x = c % d[0], y = (c / d[0]) % d[1], z = c / (d[0] * d[1]);
            int ok = 1;
            int qy = ndim >= 2 ? q : 0, qz = ndim >= 3 ? q : 0;
            for (int dz = -qz; dz <= qz && ok; dz++)
                for (int dy = -qy; dy <= qy && ok; dy++)
                    for (int dx = -q; dx <= q && ok; dx++) {
                        int dist = (dx < 0 ? -dx : dx) + (dy < 0 ? -dy : dy) + (dz < 0 ? -dz : dz);
                        if (dist == 0 || dist > q) continue;
                        int64_t xx = ((x + dx) % d[0] + d[0]) % d[0];
                        int64_t yy = ((y + dy) % d[1] + d[1]) % d[1];
                        int64_t zz = ((z + dz) % d[2] + d[2]) % d[2];
                        int64_t nb = (zz * d[1] + yy) * d[0] + xx;
                        if (nb != c && !(t[c] < t[nb] || (t[c] == t[nb] && c < nb))) ok = 0;
                    }
            fire[c] = (unsigned char)ok;
            n0 += (uint64_t)ok;
        }
        for (int64_t c = 0; c < N; c++) {          /* commit */
            if (!fire[c]) continue;
            uint32_t ctr[4] = {(uint32_t)r, (uint32_t)((uint64_t)c & 0xffffffffu), (uint32_t)((uint64_t)c >> 32), 2u}, w[4];
            oracle_philox4x32_10(ctr, key, w);
            t[c] += oracle_delta_law(w[1], w[2], inv, 0, law);
        }
        if (fired_per_round) fired_per_round[r] = n0;
    }
    if (t_out) memcpy(t_out, t, (size_t)N * 8);
    free(t); free(fire);
    return 0;
}

/* ---------------------------------------------------------------- aggregated Poisson stream
 * fig:amcpoi: the 2-D torus is partitioned into m x m subarrays C (m a power
 * of two dividing both sides; C = Y (nx/m) + X). Each C carries ONE Poisson stream of rate
 * lambda m^2 (the sum of its cells' streams); at each arrival a cell of C is
 * chosen uniformly at random (Step 2) and updated (Step 4), and T(C) advances by
 * -ln r / (lambda m^2) (Step 5). docs/PRIMITIVES.md P8: the k-th arrival of C uses Philox ctr
 * (k, C_lo, C_hi, tag_e): w0 = flip uniform (P4), (w1, w2) = the increment NLOG-2((w1 << 32) |
 * w2) at INV = floor(2^32 / (lambda m^2) + 0.5), at least 1, w3 = the cell choice
 * l = w3 >> (32 - log2 m^2) (l = 0 for m = 1; local index l = j m + i). T0(C) comes from ctr
 * (0, C_lo, C_hi, tag_i) the same way. Tags: (tag_e, tag_i) = (3, 4), except (0, 1) for m = 1,
 * where C = c and the algorithm IS fig:a1c1pe with the per-cell streams of P1 (the special
 * case pins this code to the main oracle bit for bit). Spins start from P5. The serial
 * definition: process arrivals in increasing (T(C), C) order while T(C) < T (a heap over
 * subarrays). The trajectory depends on m and is unique for a given m.
 * Event hash: P7 with ^ (l << 1) added (l = 0 for m = 1). Test infrastructure only.
 * Returns 0, -1 on bad arguments. */
typedef struct { uint64_t T; int64_t C; } agg_key;

static int agg_less(const uint64_t* T, int64_t a, int64_t b) { return T[a] < T[b] || (T[a] == T[b] && a < b); }

static void agg_sift(uint32_t* H, int64_t n, const uint64_t* T, int64_t i) {
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < n && agg_less(T, H[l], H[m])) m = l;
        if (r < n && agg_less(T, H[r], H[m])) m = r;
        if (m == i) return;
        uint32_t tmp = H[i]; H[i] = H[m]; H[m] = tmp;
        i = m;
    }
}

static uint64_t agg_delta(uint32_t w1, uint32_t w2, uint64_t inv) {
    uint64_t q = oracle_nlog_q32(((uint64_t)w1 << 32) | w2);
    uint64_t d = (uint64_t)(((unsigned __int128)q * inv) >> 32);
    return d < 1 ? 1 : d;
}

int oracle_agg_run(const int64_t* dims, int m, double lambda, double beta, double J, double h, int rule,
                   uint64_t seed, double init_q, uint64_t T_q32, int8_t* spins_out, uint64_t* T_out,
                   uint32_t* n_out, oracle_stats* st) {
    int64_t nx = dims[0], ny = dims[1];
    if (m < 1 || m > 32 || nx % m || ny % m || nx < 2 || ny < 2) return -1;
    if (!(lambda > 0) || !(beta >= 0) || (rule != 0 && rule != 1)) return -1;
    const uint64_t mm = (uint64_t)m * (uint64_t)m;
    const uint32_t tag_e = m == 1 ? 0u : 3u, tag_i = m == 1 ? 1u : 4u;
    int64_t mx = nx / m, my = ny / m, NC = mx * my, N = nx * ny;
    uint64_t thr[14];
    oracle_flip_table(2, beta, J, h, rule, thr);
    uint64_t inv = (uint64_t)floor(4294967296.0 / (lambda * (double)(m * m)) + 0.5);
    uint64_t thr_init = (uint64_t)floor(init_q * 4294967296.0);
    uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    int8_t* s = (int8_t*)malloc((size_t)N);
    uint64_t* T = (uint64_t*)malloc((size_t)NC * 8);
    uint32_t* n = (uint32_t*)calloc((size_t)NC, 4);
    uint32_t* H = (uint32_t*)malloc((size_t)NC * 4);
    if (!s || !T || !n || !H) { free(s); free(T); free(n); free(H); return -1; }
    for (int64_t c = 0; c < N; c++) {                       /* P5 spins */
        uint32_t ctr[4] = {0, (uint32_t)((uint64_t)c & 0xffffffffu), (uint32_t)((uint64_t)c >> 32), 1u}, w[4];
        oracle_philox4x32_10(ctr, key, w);
        s[c] = ((uint64_t)w[0] < thr_init) ? -1 : 1;
    }
    for (int64_t C = 0; C < NC; C++) {
        uint32_t ctr[4] = {0, (uint32_t)((uint64_t)C & 0xffffffffu), (uint32_t)((uint64_t)C >> 32), tag_i}, w[4];
        oracle_philox4x32_10(ctr, key, w);
        T[C] = agg_delta(w[1], w[2], inv);
        H[C] = (uint32_t)C;
    }
    for (int64_t i = NC / 2 - 1; i >= 0; i--) agg_sift(H, NC, T, i);
    uint64_t arrivals = 0, flips = 0, hash = 0;
    while (NC > 0) {
        int64_t C = H[0];
        if (T[C] >= T_q32) break;
        uint32_t k = n[C];
        uint32_t ctr[4] = {k, (uint32_t)((uint64_t)C & 0xffffffffu), (uint32_t)((uint64_t)C >> 32), tag_e}, w[4];
        oracle_philox4x32_10(ctr, key, w);
        int64_t l = (int64_t)(((uint64_t)w[3] * mm) >> 32);       /* Step 2: uniform cell of C (P8) */
        int64_t X = C % mx, Y = C / mx;
        int64_t x = X * m + l % m, y = Y * m + l / m;
        int64_t c = y * nx + x;
        int sigma = s[y * nx + (x + nx - 1) % nx] + s[y * nx + (x + 1) % nx] + s[((y + ny - 1) % ny) * nx + x] +
                    s[((y + 1) % ny) * nx + x];
        int sc = s[c];
        int idx = (sigma + 4) / 2 + 5 * (sc + 1) / 2;
        int ns = sc;
        if ((uint64_t)w[0] < thr[idx]) { ns = -sc; flips++; }   /* Step 4 */
        s[c] = (int8_t)ns;
        hash += oracle_ev_hash(w[3], T[C], (uint64_t)l, ns);
        T[C] += agg_delta(w[1], w[2], inv);                   /* Step 5 */
        n[C] = k + 1;
        arrivals++;
        agg_sift(H, NC, T, 0);
    }
    if (spins_out) memcpy(spins_out, s, (size_t)N);
    if (T_out) memcpy(T_out, T, (size_t)NC * 8);
    if (n_out) memcpy(n_out, n, (size_t)NC * 4);
    if (st) {
        memset(st, 0, sizeof *st);
        st->arrivals = arrivals; st->flips = flips; st->event_hash = hash;
        int64_t B = 0, M = 0;
        for (int64_t y = 0; y < ny; y++)
            for (int64_t x = 0; x < nx; x++) {
                int v = s[y * nx + x];
                M += v;
                B += v * (s[y * nx + (x + 1) % nx] + s[((y + 1) % ny) * nx + x]);
            }
        st->bond_sum = B; st->magnetisation = M;
    }
    free(s); free(T); free(n); free(H);
    return 0;
}

/* ---------------------------------------------------------------- modified BKL (P9)
 * every m x m subarray (2 <= m <= 32) of the 2-D torus runs the BKL
 * n-fold way on its kernel (the (m-2) x (m-2) interior) and the standard procedure on its
 * boundary layer Gamma_0 (fixed class, weight |Gamma_0|, may or may not change; waits for the
 * neighbouring subarrays like fig:amcpoi). Kernel classes Gamma_k are the P4 table indices
 * k = idx(s, Sigma) with integer weights W_k = |Gamma_k| thr_k (thr_k = 2^32 p_k); W_0 =
 * |Gamma_0| 2^32; W = W_0 + sum W_k. Iteration n of C: (w0..w3) = Philox ctr (n, C, 0, 5);
 * u = floor(((w0 << 32) | w1) W / 2^64). u < W_0: boundary cell number u >> 32 (increasing local
 * index l), flip iff (u & 0xffffffff) < thr[idx]. Otherwise o = u - W_0 selects class k (in
 * order 0..9) and its cell number o / thr_k (increasing l); that cell flips. The next event
 * time: T(C) += max(1, (NLOG-2((w2 << 32) | w3) INV) >> 32), INV = floor(2^64 / (lambda W') +
 * 0.5) in IEEE double, W' = the total weight AFTER the event (the new configuration holds until
 * the next event: the waiting time uses its rates). T0(C) uses ctr (0, C, 0, 6) and the initial
 * W. Spins start from P5. Serial definition: events in increasing (T(C), C) order while
 * T(C) < T. Event hash as P8 (l mixed in). Test infrastructure only. 0, or -1 on bad args. */
static uint64_t bkl_weights(const int8_t* s, int64_t nx, int64_t ny, int64_t X, int64_t Y, int m,
                            const uint64_t* thr, int* cls /* [m*m], -1 for the boundary layer */) {
    uint64_t W = 0;
    for (int l = 0; l < m * m; l++) {
        int i = l % m, j = l / m;
        if (i == 0 || j == 0 || i == m - 1 || j == m - 1) { cls[l] = -1; W += 1ULL << 32; continue; }
        int64_t x = X * m + i, y = Y * m + j;
        int sig = s[y * nx + x - 1] + s[y * nx + x + 1] + s[(y - 1) * nx + x] + s[(y + 1) * nx + x];
        int sc = s[y * nx + x];
        int k = (sig + 4) / 2 + 5 * (sc + 1) / 2;
        cls[l] = k;
        W += thr[k];
    }
    (void)ny;
    return W;
}

static uint64_t bkl_delta(uint32_t w2, uint32_t w3, double lambda, uint64_t W) {
    uint64_t q = oracle_nlog_q32(((uint64_t)w2 << 32) | w3);
    uint64_t inv = (uint64_t)floor(18446744073709551616.0 / (lambda * (double)W) + 0.5);
    uint64_t d = (uint64_t)(((unsigned __int128)q * inv) >> 32);
    return d < 1 ? 1 : d;
}

int oracle_bkl_run(const int64_t* dims, int m, double lambda, double beta, double J, double h, int rule,
                   uint64_t seed, double init_q, uint64_t T_q32, int8_t* spins_out, uint64_t* T_out,
                   uint32_t* n_out, oracle_stats* st) {
    int64_t nx = dims[0], ny = dims[1];
    if (m < 2 || m > 32 || nx % m || ny % m || nx < 2 || ny < 2) return -1;
    if (!(lambda > 0) || !(beta >= 0) || (rule != 0 && rule != 1)) return -1;
    int64_t mx = nx / m, my = ny / m, NC = mx * my, N = nx * ny;
    uint64_t thr[14];
    oracle_flip_table(2, beta, J, h, rule, thr);
    uint64_t thr_init = (uint64_t)floor(init_q * 4294967296.0);
    uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    int8_t* s = (int8_t*)malloc((size_t)N);
    uint64_t* T = (uint64_t*)malloc((size_t)NC * 8);
    uint32_t* n = (uint32_t*)calloc((size_t)NC, 4);
    uint32_t* H = (uint32_t*)malloc((size_t)NC * 4);
    int cls[1024];
    if (!s || !T || !n || !H) { free(s); free(T); free(n); free(H); return -1; }
    for (int64_t c = 0; c < N; c++) {
        uint32_t ctr[4] = {0, (uint32_t)((uint64_t)c & 0xffffffffu), (uint32_t)((uint64_t)c >> 32), 1u}, w[4];
        oracle_philox4x32_10(ctr, key, w);
        s[c] = ((uint64_t)w[0] < thr_init) ? -1 : 1;
    }
    for (int64_t C = 0; C < NC; C++) {
        uint32_t ctr[4] = {0, (uint32_t)((uint64_t)C & 0xffffffffu), (uint32_t)((uint64_t)C >> 32), 6u}, w[4];
        oracle_philox4x32_10(ctr, key, w);
        uint64_t W = bkl_weights(s, nx, ny, C % mx, C / mx, m, thr, cls);
        T[C] = bkl_delta(w[2], w[3], lambda, W);
        H[C] = (uint32_t)C;
    }
    for (int64_t i = NC / 2 - 1; i >= 0; i--) agg_sift(H, NC, T, i);
    uint64_t arrivals = 0, flips = 0, hash = 0;
    while (NC > 0) {
        int64_t C = H[0];
        if (T[C] >= T_q32) break;
        int64_t X = C % mx, Y = C / mx;
        uint32_t k = n[C];
        uint32_t ctr[4] = {k, (uint32_t)((uint64_t)C & 0xffffffffu), (uint32_t)((uint64_t)C >> 32), 5u}, w[4];
        oracle_philox4x32_10(ctr, key, w);
        uint64_t W = bkl_weights(s, nx, ny, X, Y, m, thr, cls);
        uint64_t Xr = ((uint64_t)w[0] << 32) | w[1];
        uint64_t u = (uint64_t)(((unsigned __int128)Xr * W) >> 64);
        uint64_t W0 = (uint64_t)(4 * m - 4) << 32;
        int l = -1, ns = 0;
        if (u < W0) {                                   /* boundary layer: the standard model */
            uint64_t b = u >> 32, rem = u & 0xffffffffULL, cnt = 0;
            for (int q = 0; q < m * m; q++)
                if (cls[q] < 0 && cnt++ == b) { l = q; break; }
            int64_t x = X * m + l % m, y = Y * m + l / m;
            int sig = s[y * nx + (x + nx - 1) % nx] + s[y * nx + (x + 1) % nx] + s[((y + ny - 1) % ny) * nx + x] +
                      s[((y + 1) % ny) * nx + x];
            int sc = s[y * nx + x];
            int idx = (sig + 4) / 2 + 5 * (sc + 1) / 2;
            ns = sc;
            if (rem < thr[idx]) { ns = -sc; flips++; }
            s[y * nx + x] = (int8_t)ns;
        } else {                                        /* kernel: BKL, the selected cell flips */
            uint64_t o = u - W0;
            int kc = 0;
            for (; kc < 10; kc++) {
                uint64_t cntk = 0;
                for (int q = 0; q < m * m; q++) cntk += (cls[q] == kc);
                uint64_t Wk = cntk * thr[kc];
                if (o < Wk) break;
                o -= Wk;
            }
            uint64_t r = o / thr[kc], cnt = 0;
            for (int q = 0; q < m * m; q++)
                if (cls[q] == kc && cnt++ == r) { l = q; break; }
            int64_t x = X * m + l % m, y = Y * m + l / m;
            ns = -s[y * nx + x];
            s[y * nx + x] = (int8_t)ns;
            flips++;
        }
        hash += oracle_ev_hash(w[3], T[C], (uint64_t)l, ns);
        uint64_t W2 = bkl_weights(s, nx, ny, X, Y, m, thr, cls);
        T[C] += bkl_delta(w[2], w[3], lambda, W2);
        n[C] = k + 1;
        arrivals++;
        agg_sift(H, NC, T, 0);
    }
    if (spins_out) memcpy(spins_out, s, (size_t)N);
    if (T_out) memcpy(T_out, T, (size_t)NC * 8);
    if (n_out) memcpy(n_out, n, (size_t)NC * 4);
    if (st) {
        memset(st, 0, sizeof *st);
        st->arrivals = arrivals; st->flips = flips; st->event_hash = hash;
        int64_t B = 0, M = 0;
        for (int64_t y = 0; y < ny; y++)
            for (int64_t x = 0; x < nx; x++) {
                int v = s[y * nx + x];
                M += v;
                B += v * (s[y * nx + (x + 1) % nx] + s[((y + 1) % ny) * nx + x]);
            }
        st->bond_sum = B; st->magnetisation = M;
    }
    free(s); free(T); free(n); free(H);
    return 0;
}

/* Replace the spins (user-supplied initial configuration); times and counters unchanged. */
void oracle_set_spins(oracle_sim* S, const int8_t* spins) {
    for (int64_t c = 0; c < S->N; c++) S->s[c] = spins[c] > 0 ? 1 : -1;
}
