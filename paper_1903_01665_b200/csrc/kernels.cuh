// kernels.cuh -- sm_100a device code of the fixpoint min-relaxation path.
//
// One step of the method (Algs. "SSSP: iterating over
// Points / Edges in Falcon"):  MIN(t.dist, p.dist + w(p->t), changed), i.e.
// an atomicMin on a 32-bit integer array, applied to every ACTIVE arc p->t
// until a round changes nothing.  The three processing styles differ only in
// which arcs a round visits:
//   VERTEX   -- every vertex of the CSR whose value changed in the previous
//               round (topology-driven; the activity
//               filter leaves the fixpoint unchanged, R8),
//   EDGE     -- every arc of the COO array with an active source
//               (PAPER.md:1694-1725),
//   WORKLIST -- the vertices of a frontier queue.
// BFS uses the level-synchronous update of PAPER.md:1306-1313; CC hooks
// minimum labels and pointer-jumps (reading R6).
//
// Nothing here shares code with oracle/ (DESIGN.md §4).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fk {

constexpr int32_t INF = 0x7fffffff;           // MAX_INT
constexpr uint32_t NO_STAMP = 0xffffffffu;
constexpr unsigned FULL = 0xffffffffu;

enum Algo : int { SSSP = 0, BFS = 1, CC = 2 };
enum Style : int { VERTEX = 0, EDGE = 1, WORKLIST = 2 };
enum DevStatus : int { ST_OK = 0, ST_OVERFLOW = 5, ST_NOT_CONVERGED = 6 };

// Device-resident control block: the convergence decision lives here, so no
// host round trip happens per round (replaces the per-iteration `changed`
// copy of PAPER.md:1682-1684 / SPEC.md:370).
struct Ctrl {
    uint32_t iter;        // current round, 1-based
    uint32_t in_len;      // WORKLIST: items in the input frontier
    uint32_t out_len;     // WORKLIST: items appended to the output frontier
    uint32_t changed;     // VERTEX/EDGE: some value decreased this round
    uint32_t cap;         // round cap (n + 2)
    uint32_t sel;         // WORKLIST: which buffer is the input frontier
    uint32_t done;        // fixpoint reached (or error)
    uint32_t all_active;  // WORKLIST CC round 1: frontier = all vertices (implicit)
    int32_t status;       // DevStatus
    uint32_t source;
    uint32_t pad0, pad1;
    unsigned long long launches;   // kernels launched by the fixpoint loop
    unsigned long long vertices;   // filled by k_finish
    unsigned long long edges;
    unsigned long long updates;
};

struct Args {
    uint32_t n, m;
    const uint32_t *row_off;   // [n+1]
    const uint32_t *col;       // [m]
    const int32_t *w;          // [m]
    const uint32_t *src;       // [m] COO sources (CSR order), EDGE style only
    int32_t *val;              // dist / level / label [n]
    uint32_t *stamp;           // [n] round stamps
    uint32_t *fr0, *fr1;       // frontier queues [n] each
    Ctrl *ctrl;
    unsigned long long *cnt;   // [gridDim.x * 3] per-CTA counters: vertices, edges, updates
};

// ------------------------------------------------------------------ loads
__device__ __forceinline__ uint32_t ld_ro(const uint32_t *p) { return __ldg(p); }
__device__ __forceinline__ int32_t ld_ro(const int32_t *p) { return __ldg(p); }
__device__ __forceinline__ uint4 ld_ro4(const uint32_t *p) { return __ldg(reinterpret_cast<const uint4 *>(p)); }
__device__ __forceinline__ int4 ld_ro4(const int32_t *p) { return __ldg(reinterpret_cast<const int4 *>(p)); }
// Streamed once per round: evict-first so the gathered value array keeps L2.
__device__ __forceinline__ uint32_t ld_stream(const uint32_t *p) { return __ldcs(p); }
__device__ __forceinline__ int32_t ld_stream(const int32_t *p) { return __ldcs(p); }
__device__ __forceinline__ uint4 ld_stream4(const uint32_t *p) { return __ldcs(reinterpret_cast<const uint4 *>(p)); }
__device__ __forceinline__ int4 ld_stream4(const int32_t *p) { return __ldcs(reinterpret_cast<const int4 *>(p)); }

// ------------------------------------------------------------------ block primitives
template <int B>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t &total, uint32_t *s_warp) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t v = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(FULL, v, o);
        if (lane >= o) v += y;
    }
    if (lane == 31) s_warp[wid] = v;
    __syncthreads();
    if (wid == 0) {
        uint32_t t = lane < B / 32 ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(FULL, t, o);
            if (lane >= o) t += y;
        }
        if (lane < B / 32) s_warp[lane] = t;
    }
    __syncthreads();
    total = s_warp[B / 32 - 1];
    return (wid ? s_warp[wid - 1] : 0) + v - x;
}

// Warp-aggregated frontier append: one atomicAdd per warp (ballot + popc).
__device__ __forceinline__ void warp_append(bool want, uint32_t item, uint32_t *out, uint32_t *counter) {
    const unsigned mask = __ballot_sync(FULL, want);
    if (mask == 0) return;
    const int lane = threadIdx.x & 31, leader = __ffs(mask) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(counter, (uint32_t)__popc(mask));
    base = __shfl_sync(FULL, base, leader);
    if (want) out[base + __popc(mask & ((1u << lane) - 1u))] = item;
}

template <int B>
__device__ __forceinline__ void flush_counters(const Args &a, unsigned long long nv, unsigned long long ne,
                                               unsigned long long nu, bool chg, bool ovf) {
    __shared__ unsigned long long s_red[3][B / 32];
    __shared__ int s_flags;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_flags = 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        nv += __shfl_down_sync(FULL, nv, o);
        ne += __shfl_down_sync(FULL, ne, o);
        nu += __shfl_down_sync(FULL, nu, o);
    }
    __syncthreads();
    if (lane == 0) { s_red[0][wid] = nv; s_red[1][wid] = ne; s_red[2][wid] = nu; }
    if (chg) atomicOr(&s_flags, 1);
    if (ovf) atomicOr(&s_flags, 2);
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t0 = 0, t1 = 0, t2 = 0;
        for (int i = 0; i < B / 32; i++) { t0 += s_red[0][i]; t1 += s_red[1][i]; t2 += s_red[2][i]; }
        unsigned long long *c = a.cnt + 3ull * blockIdx.x;   // this CTA's private slot: no atomics
        c[0] += t0; c[1] += t1; c[2] += t2;
        if (s_flags & 1) a.ctrl->changed = 1;
        if (s_flags & 2) a.ctrl->status = ST_OVERFLOW;
    }
}

// ------------------------------------------------------------------ init (fused)
// SSSP/BFS: dist = MAX_INT, dist[source] = 0;
// CC: label[v] = v.  Also seeds the frontier and resets the control block.
template <int ALGO>
__global__ void k_init(Args a, uint32_t source, uint32_t cap, uint32_t cnt_len) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < a.n; v += stride) {
        if (ALGO == CC) {
            a.val[v] = (int32_t)v;
            a.stamp[v] = NO_STAMP;
        } else {
            a.val[v] = v == source ? 0 : INF;
            a.stamp[v] = v == source ? 0u : NO_STAMP;
        }
    }
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt_len; i += stride) a.cnt[i] = 0ull;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        Ctrl *c = a.ctrl;
        c->iter = 1;
        c->in_len = ALGO == CC ? a.n : 1u;
        c->out_len = 0; c->changed = 0; c->cap = cap; c->sel = 0; c->done = 0;
        c->all_active = ALGO == CC ? 1u : 0u;
        c->status = ST_OK; c->source = source;
        c->launches = 1; c->vertices = 0; c->edges = 0; c->updates = 0;
        if (ALGO != CC) a.fr0[0] = source;
    }
}

// ------------------------------------------------------------------ expansion (VERTEX / WORKLIST)
// A CTA takes a tile of B*IPT items (vertices or frontier entries), each
// thread IPT consecutive ones; active items contribute their out-degree, a
// block scan turns degrees into offsets, and the CTA then walks the tile's
// concatenated arc ranges B*U arcs at a time, each thread finding its item by
// binary search in shared memory.  Every arc gets one thread regardless of
// the degree distribution (cooperative expansion for skewed RMAT degrees,
// PAPER.md:441-446), and consecutive threads read consecutive col/w words.
template <int ALGO, int STYLE, int B, int IPT, int U>
__global__ void __launch_bounds__(B) k_expand(Args a) {
    static_assert(STYLE == VERTEX || STYLE == WORKLIST, "expand is for VERTEX/WORKLIST");
    constexpr int TILE = B * IPT;
    Ctrl *c = a.ctrl;
    if (c->done) return;
    const uint32_t iter = c->iter;
    const uint32_t lev = iter - 1;   // BFS level being expanded
    uint32_t nitems;
    const uint32_t *in = nullptr;
    uint32_t *out = nullptr;
    bool implicit = STYLE == VERTEX;
    if (STYLE == WORKLIST) {
        nitems = c->in_len;
        in = c->sel ? a.fr1 : a.fr0;
        out = c->sel ? a.fr0 : a.fr1;
        implicit = c->all_active != 0;
    } else {
        nitems = a.n;
    }

    __shared__ uint32_t s_off[TILE], s_beg[TILE], s_pay[TILE], s_u[TILE];
    __shared__ uint32_t s_warp[B / 32];
    unsigned long long nv = 0, ne = 0, nu = 0;
    bool chg = false, ovf = false;

    for (uint32_t tb = blockIdx.x * TILE; tb < nitems; tb += gridDim.x * TILE) {
        uint32_t deg[IPT], beg[IPT], pay[IPT], uu[IPT];
        uint32_t sum = 0;
        const uint32_t i0 = tb + threadIdx.x * IPT;
#pragma unroll
        for (int j = 0; j < IPT; j++) {
            const uint32_t idx = i0 + j;
            deg[j] = 0; beg[j] = 0; pay[j] = 0; uu[j] = 0;
            if (idx < nitems) {
                const uint32_t u = implicit ? idx : in[idx];
                uu[j] = u;
                bool act;
                uint32_t p = 0;
                if (ALGO == SSSP) {
                    act = STYLE == WORKLIST || a.stamp[u] == iter - 1;
                    if (act) { p = (uint32_t)a.val[u]; act = p != (uint32_t)INF; }
                } else if (ALGO == BFS) {
                    act = STYLE == WORKLIST || a.val[u] == (int32_t)lev;
                } else {
                    act = true;
                    p = (uint32_t)a.val[u];   // root label after the previous compress
                }
                if (act) {
                    const uint32_t b0 = ld_ro(a.row_off + u), b1 = ld_ro(a.row_off + u + 1);
                    beg[j] = b0; deg[j] = b1 - b0; pay[j] = p;
                    nv++;
                }
            }
            sum += deg[j];
        }
        uint32_t total;
        uint32_t run = block_excl_scan<B>(sum, total, s_warp);
#pragma unroll
        for (int j = 0; j < IPT; j++) {
            const int s = threadIdx.x * IPT + j;
            s_off[s] = run; s_beg[s] = beg[j]; s_pay[s] = pay[j]; s_u[s] = uu[j];
            run += deg[j];
        }
        __syncthreads();
        if (threadIdx.x == 0) ne += total;

        for (uint32_t base = 0; base < total; base += B * U) {
            uint32_t e[U], it[U];
            bool ok[U];
#pragma unroll
            for (int q = 0; q < U; q++) {
                const uint32_t k = base + q * B + threadIdx.x;
                ok[q] = k < total;
                it[q] = 0; e[q] = 0;
                if (ok[q]) {   // largest i with s_off[i] <= k
                    int lo = 0, hi = TILE - 1;
#pragma unroll
                    for (int step = 0; step < 16; step++) {
                        if (lo >= hi) break;
                        const int mid = (lo + hi + 1) >> 1;
                        if (s_off[mid] <= k) lo = mid; else hi = mid - 1;
                    }
                    it[q] = lo;
                    e[q] = s_beg[lo] + (k - s_off[lo]);
                }
            }
            uint32_t v[U];
            int32_t wt[U];
#pragma unroll
            for (int q = 0; q < U; q++) {
                v[q] = 0; wt[q] = 0;
                if (ok[q]) {
                    v[q] = ld_stream(a.col + e[q]);
                    if (ALGO == SSSP) wt[q] = ld_stream(a.w + e[q]);
                }
            }
            int32_t cur[U];
#pragma unroll
            for (int q = 0; q < U; q++) cur[q] = ok[q] ? a.val[v[q]] : 0;
#pragma unroll
            for (int q = 0; q < U; q++) {
                bool want = false;
                uint32_t item = 0;
                if (ok[q]) {
                    if (ALGO == SSSP) {
                        const uint32_t cand = s_pay[it[q]] + (uint32_t)wt[q];
                        if (cand >= (uint32_t)INF) {
                            ovf = true;
                        } else if ((int32_t)cand < cur[q]) {
                            const int32_t old = atomicMin(a.val + v[q], (int32_t)cand);
                            if ((int32_t)cand < old) {
                                nu++;
                                if (STYLE == WORKLIST) {
                                    if (a.stamp[v[q]] != iter && atomicExch(a.stamp + v[q], iter) != iter) {
                                        want = true; item = v[q];
                                    }
                                } else {
                                    a.stamp[v[q]] = iter;
                                    chg = true;
                                }
                            }
                        }
                    } else if (ALGO == BFS) {
                        if (STYLE == WORKLIST) {
                            if (cur[q] == INF && atomicCAS(a.val + v[q], INF, (int32_t)(lev + 1)) == INF) {
                                nu++; want = true; item = v[q];
                            }
                        } else if (cur[q] > (int32_t)(lev + 1)) {   // PAPER.md:1308-1310, plain store
                            a.val[v[q]] = (int32_t)(lev + 1);
                            nu++; chg = true;
                        }
                    } else {   // CC: hook the larger root under the smaller (min-label)
                        const uint32_t lu = s_pay[it[q]], lv = (uint32_t)cur[q];
                        if (lu != lv) {
                            const uint32_t hi = lu > lv ? lu : lv, lo = lu > lv ? lv : lu;
                            const int32_t old = atomicMin(a.val + hi, (int32_t)lo);
                            if ((int32_t)lo < old) { nu++; chg = true; }
                            if (STYLE == WORKLIST) {   // keep u while one of its arcs is unresolved
                                const uint32_t u = s_u[it[q]];
                                if (a.stamp[u] != iter && atomicExch(a.stamp + u, iter) != iter) {
                                    want = true; item = u;
                                }
                            }
                        }
                    }
                }
                if (STYLE == WORKLIST) warp_append(want, item, out, &c->out_len);
            }
        }
        __syncthreads();
    }
    flush_counters<B>(a, nv, ne, nu, chg, ovf);
}

// ------------------------------------------------------------------ EDGE style (COO)
// Four CSR-ordered arcs per thread per step through 16-byte loads of src,
// col and w; col/w are only fetched when one of the four sources is active.
template <int ALGO, int B>
__global__ void __launch_bounds__(B) k_edge(Args a) {
    Ctrl *c = a.ctrl;
    if (c->done) return;
    const uint32_t iter = c->iter, lev = iter - 1;
    const uint32_t m4 = a.m >> 2, tail = a.m & 3u;
    unsigned long long nv = 0, ne = 0, nu = 0;
    bool chg = false, ovf = false;
    const uint32_t stride = gridDim.x * B;
    for (uint32_t q = blockIdx.x * B + threadIdx.x; q < m4 + (tail ? 1u : 0u); q += stride) {
        const uint32_t cntq = q < m4 ? 4u : tail;
        uint32_t s[4] = {0, 0, 0, 0}, d[4] = {0, 0, 0, 0};
        int32_t ww[4] = {0, 0, 0, 0};
        if (q < m4) {
            const uint4 s4 = ld_stream4(a.src + 4ull * q);
            s[0] = s4.x; s[1] = s4.y; s[2] = s4.z; s[3] = s4.w;
        } else {
            for (uint32_t j = 0; j < cntq; j++) s[j] = ld_stream(a.src + 4ull * q + j);
        }
        bool act[4];
        uint32_t pay[4];
        bool any = false;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            act[j] = false; pay[j] = 0;
            if ((uint32_t)j < cntq) {
                if (ALGO == SSSP) {
                    // consecutive arcs share a source: these gathers hit L1
                    act[j] = a.stamp[s[j]] == iter - 1;
                    if (act[j]) { pay[j] = (uint32_t)a.val[s[j]]; act[j] = pay[j] != (uint32_t)INF; }
                } else if (ALGO == BFS) {
                    act[j] = a.val[s[j]] == (int32_t)lev;   // e.src.dist == lev (R14)
                } else {
                    act[j] = true; pay[j] = (uint32_t)a.val[s[j]];
                }
                any |= act[j];
            }
        }
        if (!any) continue;
        if (q < m4) {
            const uint4 d4 = ld_stream4(a.col + 4ull * q);
            d[0] = d4.x; d[1] = d4.y; d[2] = d4.z; d[3] = d4.w;
            if (ALGO == SSSP) {
                const int4 w4 = ld_stream4(a.w + 4ull * q);
                ww[0] = w4.x; ww[1] = w4.y; ww[2] = w4.z; ww[3] = w4.w;
            }
        } else {
            for (uint32_t j = 0; j < cntq; j++) {
                d[j] = ld_stream(a.col + 4ull * q + j);
                if (ALGO == SSSP) ww[j] = ld_stream(a.w + 4ull * q + j);
            }
        }
        int32_t cur[4];
#pragma unroll
        for (int j = 0; j < 4; j++) cur[j] = act[j] ? a.val[d[j]] : 0;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            if (!act[j]) continue;
            ne++;
            if (ALGO == SSSP) {
                const uint32_t cand = pay[j] + (uint32_t)ww[j];
                if (cand >= (uint32_t)INF) { ovf = true; continue; }
                if ((int32_t)cand < cur[j]) {
                    const int32_t old = atomicMin(a.val + d[j], (int32_t)cand);
                    if ((int32_t)cand < old) { a.stamp[d[j]] = iter; nu++; chg = true; }
                }
            } else if (ALGO == BFS) {
                if (cur[j] > (int32_t)(lev + 1)) { a.val[d[j]] = (int32_t)(lev + 1); nu++; chg = true; }
            } else {
                const uint32_t lu = pay[j], lv = (uint32_t)cur[j];
                if (lu != lv) {
                    const uint32_t hi = lu > lv ? lu : lv, lo = lu > lv ? lv : lu;
                    const int32_t old = atomicMin(a.val + hi, (int32_t)lo);
                    if ((int32_t)lo < old) { nu++; chg = true; }
                }
            }
        }
        if (ALGO != SSSP) (void)ww;
    }
    // vertices processed: count arcs' distinct sources is not tracked in EDGE style
    flush_counters<B>(a, nv, ne, nu, chg, ovf);
}

// ------------------------------------------------------------------ CC pointer jumping
// label[v] = root of v's tree (full path compression; chains strictly
// decrease because every label is <= its vertex id).
__global__ void k_compress(Args a) {
    if (a.ctrl->done) return;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < a.n; v += stride) {
        const uint32_t r0 = (uint32_t)a.val[v];
        if (r0 == v) continue;
        uint32_t r = r0, x = (uint32_t)a.val[r];
        while (x != r) { r = x; x = (uint32_t)a.val[r]; }
        if (r != r0) a.val[v] = (int32_t)r;
    }
}

// ------------------------------------------------------------------ round advance
// Decides on the device whether another round runs ("if
// (changed == 0) break" / SPEC.md:221 "worklist non-empty"), and drives the
// CUDA-graph WHILE node through cudaGraphSetConditional.
template <int STYLE>
__global__ void k_advance(Ctrl *c, cudaGraphConditionalHandle h, int in_graph, uint32_t launches_per_round) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (c->done) {
        if (in_graph) cudaGraphSetConditional(h, 0);
        return;
    }
    c->launches += launches_per_round;
    bool more = STYLE == WORKLIST ? c->out_len > 0 : c->changed != 0;
    if (c->status != ST_OK) more = false;
    if (more && c->iter >= c->cap) { c->status = ST_NOT_CONVERGED; more = false; }
    if (more) {
        c->iter++;
        c->changed = 0;
        if (STYLE == WORKLIST) {
            c->in_len = c->out_len;
            c->out_len = 0;
            c->sel ^= 1u;
            c->all_active = 0;
        }
    } else {
        c->done = 1;
    }
    if (in_graph) cudaGraphSetConditional(h, more ? 1u : 0u);
}

// Sum the per-CTA counters into the control block.
__global__ void k_finish(Args a, uint32_t nslots) {
    __shared__ unsigned long long s[3][32];
    unsigned long long t0 = 0, t1 = 0, t2 = 0;
    for (uint32_t i = threadIdx.x; i < nslots; i += blockDim.x) {
        t0 += a.cnt[3ull * i]; t1 += a.cnt[3ull * i + 1]; t2 += a.cnt[3ull * i + 2];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        t0 += __shfl_down_sync(FULL, t0, o); t1 += __shfl_down_sync(FULL, t1, o); t2 += __shfl_down_sync(FULL, t2, o);
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) { s[0][wid] = t0; s[1][wid] = t1; s[2][wid] = t2; }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long r0 = 0, r1 = 0, r2 = 0;
        for (int i = 0; i < (int)(blockDim.x / 32); i++) { r0 += s[0][i]; r1 += s[1][i]; r2 += s[2][i]; }
        a.ctrl->vertices = r0; a.ctrl->edges = r1; a.ctrl->updates = r2;
        a.ctrl->launches += 1;
    }
}

// ------------------------------------------------------------------ load-time helpers
// Validation of the caller's CSR: flags bit0 = bad offsets,
// bit1 = col >= n, bit2 = negative weight.
__global__ void k_validate(uint32_t n, uint32_t m, const uint32_t *row_off, const uint32_t *col, const int32_t *w,
                           int *flags) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int f = 0;
    for (uint64_t v = t0; v < n; v += stride)
        if (row_off[v] > row_off[v + 1]) f |= 1;
    if (t0 == 0 && (row_off[0] != 0 || row_off[n] != m)) f |= 1;
    for (uint64_t e = t0; e < m; e += stride) {
        if (col[e] >= n) f |= 2;
        if (w && w[e] < 0) f |= 4;
    }
    if (f) atomicOr(flags, f);
}

__global__ void k_fill_i32(int32_t *p, uint64_t len, int32_t x) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += stride) p[i] = x;
}

// COO sources in CSR order: src[e] = the row containing arc e (binary search
// on row_off: largest u with row_off[u] <= e).
__global__ void k_build_src(uint32_t n, uint32_t m, const uint32_t *row_off, uint32_t *src) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
        uint32_t lo = 0, hi = n - 1;
        while (lo < hi) {
            const uint32_t mid = lo + ((hi - lo + 1) >> 1);
            if (row_off[mid] <= (uint32_t)e) lo = mid; else hi = mid - 1;
        }
        src[e] = lo;
    }
}

}  // namespace fk
