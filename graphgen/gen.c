/*
 * graphgen/gen.c -- seeded synthetic input generators (shared input infrastructure).
 *
 * This module holds NO arithmetic of the method (no relaxation, no distances,
 * no labels).  It only draws graphs and lays them out as CSR, so that both the
 * oracle (oracle/) and the CUDA path (paper_1903_01665_b200/) consume the same
 * bytes.  Recipe: SURVEY.md §8(d) "Concrete synthetic inputs" / DESIGN.md §3.
 *
 *  - PRNG: xoshiro256** seeded by splitmix64 ("splitmix64-seeded
 *    xoshiro-class generator; exact algorithm documented and frozen").
 *  - Arcs are produced in fixed chunks of 2^20; chunk c owns its own generator
 *    seeded from seed ^ (c * 0x9E3779B97F4A7C15), so the output is identical
 *    for any thread count.
 *  - Uniform [0,k): Lemire multiply-shift on the top 32 bits, with rejection.
 *  - G(n,m) (Table 1 rand-* rows): src=U[0,n),
 *    dst=U[0,n), redraw both on src==dst, then w = 1+U[0,100).
 *  - R-MAT (Table 1 rmat-* rows): L=ceil(log2 n)
 *    levels, one uniform double per level picks the quadrant; redraw the pair
 *    if an id >= n or a self loop; then w; then a Fisher-Yates relabelling.
 *  - Road-like grid (Table 1 USA-* rows, shape only): W x H lattice,
 *    each lattice edge kept with probability p, both arcs with one weight.
 *  - CSR: stable counting sort by src ("CSR edge order = stable
 *    sort by (src, input order)").
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define CHUNK_LOG 20
#define CHUNK ((uint64_t)1 << CHUNK_LOG)
#define GOLDEN 0x9E3779B97F4A7C15ull

static inline uint64_t splitmix64(uint64_t *x) {
    uint64_t z = (*x += GOLDEN);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

typedef struct { uint64_t s[4]; } xo_t;

static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

static inline uint64_t xo_next(xo_t *r) {
    uint64_t *s = r->s;
    uint64_t result = rotl(s[1] * 5, 7) * 9;
    uint64_t t = s[1] << 17;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3];
    s[2] ^= t; s[3] = rotl(s[3], 45);
    return result;
}

static inline void xo_seed(xo_t *r, uint64_t seed) {
    uint64_t x = seed;
    for (int i = 0; i < 4; i++) r->s[i] = splitmix64(&x);
}

/* Uniform integer in [0,k), k >= 1 (Lemire multiply-shift with rejection). */
static inline uint32_t uni(xo_t *r, uint32_t k) {
    uint64_t mm = (uint64_t)(uint32_t)(xo_next(r) >> 32) * (uint64_t)k;
    uint32_t l = (uint32_t)mm;
    if (l < k) {
        uint32_t t = (uint32_t)(-k) % k;
        while (l < t) {
            mm = (uint64_t)(uint32_t)(xo_next(r) >> 32) * (uint64_t)k;
            l = (uint32_t)mm;
        }
    }
    return (uint32_t)(mm >> 32);
}

static inline double unif01(xo_t *r) { return (double)(xo_next(r) >> 11) * 0x1.0p-53; }

uint64_t gg_xoshiro_first(uint64_t seed) { xo_t r; xo_seed(&r, seed); return xo_next(&r); }
uint32_t gg_uniform_first(uint64_t seed, uint32_t k) { xo_t r; xo_seed(&r, seed); return uni(&r, k); }

/* ---------------- G(n,m) directed ---------------- */
int gg_er(uint64_t n, uint64_t m, uint64_t seed, uint32_t *src, uint32_t *dst, int32_t *w) {
    if (m > 0 && n < 2) return -1;
    if (n > 0xFFFFFFFFull) return -1;
    uint64_t nchunks = (m + CHUNK - 1) / CHUNK;
#pragma omp parallel for schedule(dynamic, 1)
    for (uint64_t c = 0; c < nchunks; c++) {
        xo_t r; xo_seed(&r, seed ^ (c * GOLDEN));
        uint64_t lo = c * CHUNK, hi = lo + CHUNK < m ? lo + CHUNK : m;
        for (uint64_t e = lo; e < hi; e++) {
            uint32_t s, d;
            do { s = uni(&r, (uint32_t)n); d = uni(&r, (uint32_t)n); } while (s == d);
            src[e] = s; dst[e] = d; w[e] = 1 + (int32_t)uni(&r, 100);
        }
    }
    return 0;
}

/* ---------------- R-MAT ---------------- */
int gg_rmat(uint64_t n, uint64_t m, uint64_t seed, double a, double b, double c, int relabel,
            uint32_t *src, uint32_t *dst, int32_t *w) {
    if (m > 0 && n < 2) return -1;
    if (n > 0xFFFFFFFFull) return -1;
    int L = 0;
    while (((uint64_t)1 << L) < n) L++;
    double ab = a + b, abc = a + b + c;
    uint64_t nchunks = (m + CHUNK - 1) / CHUNK;
#pragma omp parallel for schedule(dynamic, 1)
    for (uint64_t ch = 0; ch < nchunks; ch++) {
        xo_t r; xo_seed(&r, seed ^ (ch * GOLDEN));
        uint64_t lo = ch * CHUNK, hi = lo + CHUNK < m ? lo + CHUNK : m;
        for (uint64_t e = lo; e < hi; e++) {
            uint64_t s, d;
            for (;;) {
                s = 0; d = 0;
                for (int l = 0; l < L; l++) {
                    double x = unif01(&r);
                    uint64_t sb, db;
                    if (x < a) { sb = 0; db = 0; }
                    else if (x < ab) { sb = 0; db = 1; }
                    else if (x < abc) { sb = 1; db = 0; }
                    else { sb = 1; db = 1; }
                    s = (s << 1) | sb; d = (d << 1) | db;
                }
                if (s < n && d < n && s != d) break;
            }
            src[e] = (uint32_t)s; dst[e] = (uint32_t)d; w[e] = 1 + (int32_t)uni(&r, 100);
        }
    }
    if (relabel && n > 1) {
        uint32_t *perm = (uint32_t *)malloc(n * sizeof(uint32_t));
        if (!perm) return -2;
        for (uint64_t i = 0; i < n; i++) perm[i] = (uint32_t)i;
        xo_t r; xo_seed(&r, seed ^ 0xA5A5A5A5A5A5A5A5ull);
        for (uint64_t i = n - 1; i > 0; i--) {
            uint32_t j = uni(&r, (uint32_t)(i + 1));
            uint32_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
        }
#pragma omp parallel for schedule(static)
        for (uint64_t e = 0; e < m; e++) { src[e] = perm[src[e]]; dst[e] = perm[dst[e]]; }
        free(perm);
    }
    return 0;
}

/* ---------------- road-like 2-D grid ----------------
 * Lattice edges are indexed row-major: first the H*(W-1) horizontal edges
 * (r,c)-(r,c+1), then the (H-1)*W vertical edges (r,c)-(r+1,c).  Vertex id =
 * r*W + c.  Per lattice edge: keep-coin U32 < floor(p*2^32); if kept, draw w
 * and emit (u,v,w) then (v,u,w).  Call with src==NULL to only count arcs.   */
int64_t gg_grid(uint64_t W, uint64_t H, double p, uint64_t seed, uint32_t *src, uint32_t *dst, int32_t *w) {
    if (W * H > 0xFFFFFFFFull) return -1;
    uint64_t nh = H * (W > 0 ? W - 1 : 0), nv = (H > 0 ? H - 1 : 0) * W, ne = nh + nv;
    uint64_t thr = (uint64_t)floor(p * 4294967296.0);
    uint64_t nchunks = (ne + CHUNK - 1) / CHUNK;
    uint64_t *cnt = (uint64_t *)calloc(nchunks + 1, sizeof(uint64_t));
    if (!cnt) return -2;
    /* pass 1: count kept edges per chunk */
#pragma omp parallel for schedule(dynamic, 1)
    for (uint64_t c = 0; c < nchunks; c++) {
        xo_t r; xo_seed(&r, seed ^ (c * GOLDEN));
        uint64_t lo = c * CHUNK, hi = lo + CHUNK < ne ? lo + CHUNK : ne, k = 0;
        for (uint64_t e = lo; e < hi; e++) {
            uint64_t coin = xo_next(&r) >> 32;
            if (coin < thr) { k++; (void)uni(&r, 100); }
        }
        cnt[c + 1] = k;
    }
    for (uint64_t c = 0; c < nchunks; c++) cnt[c + 1] += cnt[c];
    int64_t total = (int64_t)(2 * cnt[nchunks]);
    if (src) {
#pragma omp parallel for schedule(dynamic, 1)
        for (uint64_t c = 0; c < nchunks; c++) {
            xo_t r; xo_seed(&r, seed ^ (c * GOLDEN));
            uint64_t lo = c * CHUNK, hi = lo + CHUNK < ne ? lo + CHUNK : ne, o = 2 * cnt[c];
            for (uint64_t e = lo; e < hi; e++) {
                uint64_t coin = xo_next(&r) >> 32;
                if (coin < thr) {
                    int32_t wt = 1 + (int32_t)uni(&r, 100);
                    uint64_t u, v;
                    if (e < nh) { uint64_t row = e / (W - 1), col = e % (W - 1); u = row * W + col; v = u + 1; }
                    else { uint64_t f = e - nh; u = f; v = f + W; }
                    src[o] = (uint32_t)u; dst[o] = (uint32_t)v; w[o] = wt; o++;
                    src[o] = (uint32_t)v; dst[o] = (uint32_t)u; w[o] = wt; o++;
                }
            }
        }
    }
    free(cnt);
    return total;
}

/* ---------------- CSR by stable counting sort on src ---------------- */
int gg_csr(uint64_t n, uint64_t m, const uint32_t *src, const uint32_t *dst, const int32_t *w,
           uint32_t *row_off, uint32_t *col, int32_t *wout) {
    if (m > 0xFFFFFFFFull) return -1;
    memset(row_off, 0, (n + 1) * sizeof(uint32_t));
    for (uint64_t e = 0; e < m; e++) {
        if (src[e] >= n || dst[e] >= n) return -3;
        row_off[src[e] + 1]++;
    }
    for (uint64_t v = 0; v < n; v++) row_off[v + 1] += row_off[v];
    uint32_t *pos = (uint32_t *)malloc((n + 1) * sizeof(uint32_t));
    if (!pos) return -2;
    memcpy(pos, row_off, (n + 1) * sizeof(uint32_t));
    for (uint64_t e = 0; e < m; e++) {
        uint32_t p = pos[src[e]]++;
        col[p] = dst[e];
        if (w && wout) wout[p] = w[e];
    }
    free(pos);
    return 0;
}

/* Seeded source: stream seed^0x5EED, draw U[0,n) until
 * out-degree >= 1 (gives up after 64 draws + linear scan; returns 0 if m==0). */
uint32_t gg_pick_source(uint64_t n, const uint32_t *row_off, uint64_t seed) {
    if (n == 0) return 0;
    xo_t r; xo_seed(&r, seed ^ 0x5EEDull);
    for (int t = 0; t < 4096; t++) {
        uint32_t s = uni(&r, (uint32_t)n);
        if (row_off[s + 1] > row_off[s]) return s;
    }
    for (uint64_t v = 0; v < n; v++) if (row_off[v + 1] > row_off[v]) return (uint32_t)v;
    return 0;
}

int gg_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
