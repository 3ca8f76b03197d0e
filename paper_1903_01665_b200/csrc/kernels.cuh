// kernels.cuh -- sm_100a device code of the fixpoint min-relaxation path.
//
// One step of the method (Algs. "SSSP: iterating over
// Points / Edges in Falcon"):  MIN(t.dist, p.dist + w(p->t), changed), i.e.
// an atomicMin on a 32-bit integer array, applied to every ACTIVE arc p->t
// until a round changes nothing.  The three processing styles differ only in
// which arcs a round visits:
//   VERTEX   -- every vertex is visited (topology-driven, PAPER.md:1683
//               "foreach (t In graph.points)"); those whose value changed in
//               the previous round (R8) / whose level is lev (BFS,
//               PAPER.md:1322) expand their CSR row,
//   EDGE     -- every arc of the COO array with an active source
//               (PAPER.md:1694-1725),
//   WORKLIST -- the vertices of a frontier queue.
// BFS uses the level-synchronous update of PAPER.md:1306-1313; CC hooks
// minimum labels and pointer-jumps (reading R6).
//
// Activity sets are bitmaps (n bits, a few MB, L2-resident): bm[r % 3] holds
// the vertices improved in round r; round r reads bm[(r-1) % 3], writes
// bm[r % 3] and clears bm[(r+1) % 3] for the next round.  BFS also keeps a
// visited bitmap.  The value array is gathered with an L2 evict-last policy,
// the streamed CSR/COO arrays with evict-first.
//
// Nothing here shares code with oracle/ (DESIGN.md §4).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fk {

constexpr int32_t INF = 0x7fffffff;   // MAX_INT
constexpr unsigned FULL = 0xffffffffu;

enum Algo : int { SSSP = 0, BFS = 1, CC = 2 };
enum Style : int { VERTEX = 0, EDGE = 1, WORKLIST = 2 };
enum DevStatus : int { ST_OK = 0, ST_OVERFLOW = 5, ST_NOT_CONVERGED = 6 };

// Device-resident control block: the convergence decision lives here, so no
// host round trip happens per round (replaces the per-iteration `changed`
// copy of PAPER.md:1682-1684 / SPEC.md:370).
struct Ctrl {
    uint32_t iter;        // current round, 1-based
    uint32_t in_len;      // items in the input frontier (VERTEX: built by k_scan)
    uint32_t out_len;     // WORKLIST: items appended to the output frontier
    uint32_t changed;     // VERTEX/EDGE: some value decreased this round
    uint32_t cap;         // round cap (n + 2)
    uint32_t sel;         // WORKLIST: which buffer is the input frontier
    uint32_t done;        // fixpoint reached (or error)
    uint32_t all_active;  // CC round 1: frontier = all vertices (implicit)
    int32_t status;       // DevStatus
    uint32_t source;
    uint32_t pull;        // BFS VERTEX: this round runs bottom-up (pull over in-arcs)
    uint32_t found;       // BFS: vertices discovered this round (direction heuristic)
    unsigned long long launches;   // kernels launched by the fixpoint loop
    unsigned long long vertices;   // filled by k_finish
    unsigned long long edges;
    unsigned long long updates;
};

struct Args {
    uint32_t n, m, nwords;     // nwords = ceil(n / 32), rounded up to a multiple of 4
    const uint32_t *row_off;   // [n+1]
    const uint32_t *col;       // [m]
    const int32_t *w;          // [m]
    const uint2 *cw;           // [m] (col, w) interleaved: SSSP reads one 8-byte word per arc
    const uint32_t *src;       // [m] COO sources (CSR order), EDGE style only
    const uint32_t *rin_off;   // [n+1] reverse CSR (in-arcs), BFS pull only
    const uint32_t *rin_col;   // [m]
    int32_t *val;              // dist / level / label [n]
    uint32_t *bm0, *bm1, *bm2; // round bitmaps [nwords] each
    uint32_t *vis;             // BFS visited bitmap [nwords]
    uint32_t *fr0, *fr1;       // frontier queues [n] each
    Ctrl *ctrl;
    unsigned long long *cnt;   // [gridDim.x * 3] per-CTA counters: vertices, edges, updates
};

__device__ __forceinline__ uint32_t *bm_of(const Args &a, uint32_t r) {
    const uint32_t k = r % 3u;
    return k == 0 ? a.bm0 : (k == 1 ? a.bm1 : a.bm2);
}

// ------------------------------------------------------------------ loads with L2 policies
__device__ __forceinline__ uint64_t pol_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t pol_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// read-only, streamed once per round: no L1 allocation, evict-first in L2
__device__ __forceinline__ uint32_t ld_stream(const uint32_t *p, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int32_t ld_stream(const int32_t *p, uint64_t pol) {
    int32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint4 ld_stream4(const uint32_t *p, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int4 ld_stream4(const int32_t *p, uint64_t pol) {
    int4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint2 ld_stream2(const uint2 *p, uint64_t pol) {
    uint2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
                 : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint4 ld_stream4(const uint2 *p, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
    return v;
}
// mutable value array (written by atomics in the same kernel): coherent
// load, evict-last so the gathered array stays L2-resident
__device__ __forceinline__ int32_t ld_val(const int32_t *p, uint64_t pol) {
    int32_t v;
    asm volatile("ld.global.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint32_t ld_ro(const uint32_t *p) { return __ldg(p); }

__device__ __forceinline__ bool bit_test(const uint32_t *bm, uint32_t v) { return (bm[v >> 5] >> (v & 31)) & 1u; }

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
    const uint32_t r = (wid ? s_warp[wid - 1] : 0) + v - x;
    __syncthreads();   // s_warp may be reused right away
    return r;
}

template <int B>
__device__ __forceinline__ void flush_counters(const Args &a, unsigned long long nv, unsigned long long ne,
                                               unsigned long long nu, bool chg, bool ovf, bool count_found = false) {
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
        if (count_found && t2) atomicAdd(&a.ctrl->found, (uint32_t)t2);
        if (s_flags & 1) a.ctrl->changed = 1;
        if (s_flags & 2) a.ctrl->status = ST_OVERFLOW;
    }
}

// Clear the bitmap of round r+1 (grid-stride, 16-byte stores).
__device__ __forceinline__ void clear_next_bitmap(const Args &a, uint32_t r) {
    uint4 *p = reinterpret_cast<uint4 *>(bm_of(a, r + 1));
    const uint32_t n4 = a.nwords >> 2;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x)
        p[i] = make_uint4(0, 0, 0, 0);
}

// ------------------------------------------------------------------ block-level frontier queue
// Appends are staged in shared memory (warp-aggregated shared atomics) and
// written out with ONE global atomicAdd per flush: a single global counter hit
// by every warp serialises in one L2 slice.
template <int B, int QCAP>
struct BlockQueue {
    uint32_t *q;      // [QCAP] shared
    uint32_t *cnt;    // shared
    uint32_t *base;   // shared
    __device__ __forceinline__ void push(bool want, uint32_t item) {   // warp-collective
        const unsigned mask = __ballot_sync(FULL, want);
        if (mask == 0) return;
        const int lane = threadIdx.x & 31, leader = __ffs(mask) - 1;
        uint32_t b = 0;
        if (lane == leader) b = atomicAdd(cnt, (uint32_t)__popc(mask));
        b = __shfl_sync(FULL, b, leader);
        if (want) q[b + __popc(mask & ((1u << lane) - 1u))] = item;
    }
    // block-collective; flushes when more than `thresh` items are staged
    __device__ __forceinline__ void flush(uint32_t *out, uint32_t *gcounter, uint32_t thresh) {
        __syncthreads();
        const uint32_t c = *cnt;
        if (c > thresh) {
            if (threadIdx.x == 0) *base = atomicAdd(gcounter, c);
            __syncthreads();
            const uint32_t b = *base;
            for (uint32_t i = threadIdx.x; i < c; i += B) out[b + i] = q[i];
            __syncthreads();
            if (threadIdx.x == 0) *cnt = 0;
            __syncthreads();
        }
    }
};

// ------------------------------------------------------------------ init (fused)
// SSSP/BFS: dist = MAX_INT, dist[source] = 0;
// CC: label[v] = v.  Clears the bitmaps (source bit set in bm0 / vis), seeds
// the frontier and resets the control block, in one launch.
template <int ALGO>
__global__ void k_init(Args a, uint32_t source, uint32_t cap, uint32_t cnt_len, int style) {
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t t0 = blockIdx.x * blockDim.x + threadIdx.x;
    for (uint32_t v = t0; v < a.n; v += stride) {
        if (ALGO == CC) a.val[v] = (int32_t)v;
        else a.val[v] = v == source ? 0 : INF;
    }
    const uint32_t sw = ALGO == CC ? 0xffffffffu : source >> 5, sb = 1u << (source & 31);
    for (uint32_t i = t0; i < a.nwords; i += stride) {
        a.bm0[i] = i == sw ? sb : 0u;
        a.bm1[i] = 0u; a.bm2[i] = 0u;
        if (ALGO == BFS) a.vis[i] = i == sw ? sb : 0u;
    }
    for (uint32_t i = t0; i < cnt_len; i += stride) a.cnt[i] = 0ull;
    if (t0 == 0) {
        Ctrl *c = a.ctrl;
        c->iter = 1;
        c->in_len = ALGO == CC ? a.n : (style == VERTEX ? 0u : 1u);   // VERTEX: k_scan builds it
        c->out_len = 0; c->changed = 0; c->cap = cap; c->sel = 0; c->done = 0;
        c->all_active = ALGO == CC ? 1u : 0u;
        c->status = ST_OK; c->source = source;
        c->launches = 1; c->vertices = 0; c->edges = 0; c->updates = 0;
        c->pull = 0; c->found = 0;
        if (ALGO != CC) a.fr0[0] = source;
    }
}

// ------------------------------------------------------------------ VERTEX activity scan
// Topology-driven round, part 1: visit EVERY vertex through
// its bit in bm[(r-1)%3] and compact the active ones, in vertex order, into
// the frontier.  Each CTA owns a contiguous range of bitmap words: pass 1
// counts its set bits (one global atomicAdd per CTA per round), pass 2 writes
// them warp-cooperatively (one ballot per word: coalesced stores).  Also
// clears bm[(r+1)%3].
template <int ALGO, int B>
__global__ void __launch_bounds__(B) k_scan(Args a) {
    constexpr int NW = B / 32;
    Ctrl *c = a.ctrl;
    if (c->done) return;
    const uint32_t iter = c->iter, lev = iter - 1;
    clear_next_bitmap(a, iter);
    // BFS: levels are written here, in vertex order, for the vertices the
    // previous round discovered (bm[(r-1)%3]) -- dense sequential stores
    // instead of one random store per discovery.  A pull round writes the
    // levels but needs no compacted frontier.
    const bool compact = !(ALGO == BFS && c->pull);
    const uint32_t *bm = bm_of(a, iter - 1);
    __shared__ uint32_t s_w[NW];
    __shared__ uint32_t s_base;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t per = ((a.nwords + gridDim.x - 1) / gridDim.x + B - 1) / B * B;
    const uint32_t lo = blockIdx.x * per;
    const uint32_t hi = lo + per < a.nwords ? lo + per : a.nwords;
    uint32_t run = 0;
    if (compact) {   // pass 1: count (block-uniform branch)
        uint32_t cnt = 0;
        for (uint32_t i = lo + threadIdx.x; i < hi; i += B) cnt += __popc(bm[i]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(FULL, cnt, o);
        if (lane == 0) s_w[wid] = cnt;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t t = 0;
            for (int i = 0; i < NW; i++) t += s_w[i];
            s_base = t ? atomicAdd(&c->in_len, t) : 0;
        }
        __syncthreads();
        run = s_base;
        __syncthreads();
    }
    // pass 2: write, B words per CTA step, 32 words per warp
    for (uint32_t i0 = lo; i0 < hi; i0 += B) {   // block-uniform
        const uint32_t i = i0 + threadIdx.x;
        const uint32_t w = i < hi ? bm[i] : 0u;
        if (ALGO == BFS && w) {
            uint32_t x = w;
            while (x) {
                const int bp = __ffs(x) - 1;
                x &= x - 1;
                a.val[i * 32u + bp] = (int32_t)lev;
            }
        }
        if (!compact) continue;
        uint32_t incl = __popc(w);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t excl = incl - __popc(w);
        if (lane == 31) s_w[wid] = incl;
        __syncthreads();
        uint32_t wbase = run, tot = 0;
        for (int k = 0; k < NW; k++) {
            const uint32_t x = s_w[k];
            if (k < wid) wbase += x;
            tot += x;
        }
        __syncthreads();
        run += tot;
        const uint32_t wbeg = i0 + 32 * wid;
        for (int j = 0; j < 32; j++) {   // warp-uniform
            const uint32_t wj = __shfl_sync(FULL, w, j);
            if (wj == 0) continue;
            const uint32_t ej = __shfl_sync(FULL, excl, j);
            if ((wj >> lane) & 1u)
                a.fr0[wbase + ej + __popc(wj & ((1u << lane) - 1u))] = (wbeg + j) * 32u + lane;
        }
    }
}

// ------------------------------------------------------------------ BFS bottom-up (pull) round
// Direction-optimising BFS, VERTEX style over `innbrs` (Table
// "Iterators"): every unvisited vertex scans its in-arcs until it finds a
// parent in the previous level (bm[(r-1)%3]).  A warp owns one 32-vertex
// bitmap word, so the visited / next-frontier words are written with plain
// stores.  Run when the frontier is large (k_advance).
template <int B>
__global__ void __launch_bounds__(B) k_pull(Args a) {
    Ctrl *c = a.ctrl;
    if (c->done || !c->pull) return;
    const uint32_t iter = c->iter;
    const uint32_t *bm_prev = bm_of(a, iter - 1);
    uint32_t *bm_now = bm_of(a, iter);
    const int lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * B + threadIdx.x) >> 5, nwarps = (gridDim.x * B) >> 5;
    unsigned long long nv = 0, ne = 0, nu = 0;
    bool chg = false;
    for (uint32_t wi = gw; wi < a.nwords; wi += nwarps) {
        const uint32_t visw = a.vis[wi];
        const uint32_t v = wi * 32u + lane;
        bool found = false;
        if (v < a.n && !((visw >> lane) & 1u)) {
            nv++;
            const uint32_t e1 = ld_ro(a.rin_off + v + 1);
            for (uint32_t e = ld_ro(a.rin_off + v); e < e1; e++) {
                ne++;
                if (bit_test(bm_prev, ld_ro(a.rin_col + e))) { found = true; break; }
            }
        }
        const unsigned mask = __ballot_sync(FULL, found);
        if (mask && lane == 0) {
            a.vis[wi] = visw | mask;
            bm_now[wi] = mask;
        }
        if (found) { nu++; chg = true; }
    }
    flush_counters<B>(a, nv, ne, nu, chg, false, true);
}

// ------------------------------------------------------------------ expansion (VERTEX / WORKLIST)
// A CTA takes a tile of B*IPT items (frontier entries, or all vertices for
// CC), each thread IPT consecutive ones; active items contribute their
// out-degree, a block scan turns degrees into offsets, and the CTA then walks
// the tile's concatenated arc ranges B*U arcs at a time, each thread finding
// its item by binary search in shared memory.  Every arc gets one thread
// regardless of the degree distribution (cooperative expansion for skewed
// RMAT degrees), and consecutive threads read consecutive
// col/w words.
//   VERTEX  : items = the frontier k_scan compacted (CC: all vertices);
//             an improvement marks v in bm[r%3] / sets `changed`.
//   WORKLIST: items = the queue of the previous round; an improvement appends
//             v once per round (bitmap claim).
template <int ALGO, int STYLE, int B, int IPT, int U>
__global__ void __launch_bounds__(B, 4) k_expand(Args a) {
    static_assert(STYLE == VERTEX || STYLE == WORKLIST, "expand is for VERTEX/WORKLIST");
    constexpr int TILE = B * IPT;
    constexpr int QCAP = STYLE == WORKLIST ? 2 * B * U : 1;
    Ctrl *c = a.ctrl;
    if (c->done) return;
    const uint32_t iter = c->iter;
    const uint32_t lev = iter - 1;   // BFS level being expanded
    const uint32_t *in = c->sel ? a.fr1 : a.fr0;
    uint32_t *out = c->sel ? a.fr0 : a.fr1;
    const bool implicit = ALGO == CC && (STYLE == VERTEX || c->all_active != 0);
    const uint32_t nitems = implicit ? a.n : c->in_len;
    uint32_t *bm_now = bm_of(a, iter);
    if (STYLE == WORKLIST || ALGO == CC) clear_next_bitmap(a, iter);   // VERTEX SSSP/BFS: k_scan clears
    const uint64_t pf = pol_evict_first(), pl = pol_evict_last();

    __shared__ uint32_t s_off[TILE], s_beg[TILE], s_pay[TILE], s_u[TILE];
    __shared__ uint32_t s_warp[B / 32];
    __shared__ uint32_t s_q[QCAP];
    __shared__ uint32_t s_cnt, s_base;
    if (threadIdx.x == 0) s_cnt = 0;
    BlockQueue<B, QCAP> bq{s_q, &s_cnt, &s_base};
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
                const uint32_t u = implicit ? idx : ld_stream(in + idx, pf);
                uu[j] = u;
                bool act = true;
                uint32_t p = 0;
                if (ALGO == SSSP) {
                    p = (uint32_t)ld_val(a.val + u, pl);
                    act = p != (uint32_t)INF;
                } else if (ALGO == CC) {
                    p = (uint32_t)ld_val(a.val + u, pl);   // root label after the previous compress
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
                    if (ALGO == SSSP) {   // one 8-byte (col, w) word: one DRAM burst per row
                        const uint2 x = ld_stream2(a.cw + e[q], pf);
                        v[q] = x.x; wt[q] = (int32_t)x.y;
                    } else {
                        v[q] = ld_stream(a.col + e[q], pf);
                    }
                }
            }
            int32_t cur[U];
#pragma unroll
            for (int q = 0; q < U; q++) {
                cur[q] = 0;
                if (ok[q]) {
                    if (ALGO == BFS) cur[q] = bit_test(a.vis, v[q]) ? 0 : INF;   // visited filter
                    else cur[q] = ld_val(a.val + v[q], pl);
                }
            }
            // Phased so that the U arcs' dependent round trips overlap:
            // (D) the atomics whose old value decides the outcome, (E) the
            // bitmap claims, (F) the queue pushes.
            int32_t old[U];
            uint32_t key[U];   // SSSP: cand; CC: lo; BFS: unused
            bool tried[U];
#pragma unroll
            for (int q = 0; q < U; q++) {
                tried[q] = false; old[q] = 0; key[q] = 0;
                if (!ok[q]) continue;
                if (ALGO == SSSP) {
                    const uint32_t cand = s_pay[it[q]] + (uint32_t)wt[q];
                    key[q] = cand;
                    if (cand >= (uint32_t)INF) {
                        ovf = true;
                    } else if ((int32_t)cand < cur[q]) {
                        old[q] = atomicMin(a.val + v[q], (int32_t)cand);
                        tried[q] = true;
                    }
                } else if (ALGO == BFS) {
                    // t.dist > lev+1 -> t.dist = lev+1; the visited
                    // claim makes the store (and the append) happen exactly once
                    if (cur[q] == INF) {
                        old[q] = (int32_t)atomicOr(a.vis + (v[q] >> 5), 1u << (v[q] & 31));
                        tried[q] = true;
                    }
                } else {   // CC: hook the larger root under the smaller (min-label)
                    const uint32_t lu = s_pay[it[q]], lv = (uint32_t)cur[q];
                    if (lu != lv) {
                        const uint32_t hi = lu > lv ? lu : lv, lo = lu > lv ? lv : lu;
                        key[q] = lo;
                        old[q] = atomicMin(a.val + hi, (int32_t)lo);
                        tried[q] = true;
                    }
                }
            }
            bool need[U];
            uint32_t citem[U];
#pragma unroll
            for (int q = 0; q < U; q++) {
                need[q] = false; citem[q] = 0;
                if (!tried[q]) continue;
                if (ALGO == SSSP) {
                    if ((int32_t)key[q] < old[q]) { nu++; chg = true; need[q] = true; citem[q] = v[q]; }
                } else if (ALGO == BFS) {
                    if (!((uint32_t)old[q] & (1u << (v[q] & 31)))) {
                        a.val[v[q]] = (int32_t)(lev + 1);
                        nu++; chg = true;
                        if (STYLE == WORKLIST) { need[q] = true; citem[q] = v[q]; }
                        else atomicOr(bm_now + (v[q] >> 5), 1u << (v[q] & 31));
                    }
                } else {
                    if ((int32_t)key[q] < old[q]) { nu++; chg = true; }
                    if (STYLE == WORKLIST) { need[q] = true; citem[q] = s_u[it[q]]; }   // keep u while unresolved
                }
            }
            uint32_t got[U];
#pragma unroll
            for (int q = 0; q < U; q++) {
                got[q] = 0xffffffffu;
                if (!need[q]) continue;
                if (ALGO == BFS) { got[q] = 0; continue; }   // the visited claim was the dedup
                const uint32_t b = 1u << (citem[q] & 31);
                if (STYLE == WORKLIST) got[q] = atomicOr(bm_now + (citem[q] >> 5), b);
                else atomicOr(bm_now + (citem[q] >> 5), b);   // no return value: a reduction
            }
            if (STYLE == WORKLIST) {
#pragma unroll
                for (int q = 0; q < U; q++)
                    bq.push(need[q] && !(got[q] & (1u << (citem[q] & 31))), citem[q]);
            }
            if (STYLE == WORKLIST) bq.flush(out, &c->out_len, QCAP > B * U ? QCAP - B * U : 0);
        }
        __syncthreads();
    }
    if (STYLE == WORKLIST) bq.flush(out, &c->out_len, 0);
    flush_counters<B>(a, nv, ne, nu, chg, ovf);
}

// ------------------------------------------------------------------ warp-centric expansion
// Same work as k_expand, but a WARP owns 32 items: a shuffle scan turns their
// degrees into offsets and the warp walks the concatenated arc ranges 32*U
// arcs at a time, each lane finding its item by a 5-step shuffle binary
// search.  No block barrier in the loop, so warps drift freely.  The path is
// bound by the latency of dependent memory round trips, so:
//  * item loads are software-pipelined two tiles ahead (frontier entry two
//    tiles ahead, value / row offsets one tile ahead);
//  * VERTEX relaxations are fire-and-forget: the read filter `cand < val[v]`
//    decides, atomicMin / the bitmap OR are issued as reductions (RED) whose
//    results nobody waits for.  A vertex whose read passed the filter is
//    improved in this round -- by us, or by whoever lowered it further after
//    our read, who marks it too -- so the marked set is exactly the set of
//    vertices improved this round (R8);
//  * WORKLIST needs the old bitmap word to append each vertex once.
template <int ALGO, int STYLE, int B, int U, int MINB>
__global__ void __launch_bounds__(B, MINB) k_expand_warp(Args a) {
    static_assert(STYLE == VERTEX || STYLE == WORKLIST, "expand is for VERTEX/WORKLIST");
    constexpr int NW = B / 32;
    constexpr int WQ = STYLE == WORKLIST ? 512 : 1;
    Ctrl *c = a.ctrl;
    if (c->done || (ALGO == BFS && STYLE == VERTEX && c->pull)) return;
    const uint32_t iter = c->iter;
    const uint32_t lev = iter - 1;
    const uint32_t *in = c->sel ? a.fr1 : a.fr0;
    uint32_t *out = c->sel ? a.fr0 : a.fr1;
    const bool implicit = ALGO == CC && (STYLE == VERTEX || c->all_active != 0);
    const uint32_t nitems = implicit ? a.n : c->in_len;
    uint32_t *bm_now = bm_of(a, iter);
    if (STYLE == WORKLIST || ALGO == CC) clear_next_bitmap(a, iter);
    const uint64_t pf = pol_evict_first(), pl = pol_evict_last();

    __shared__ uint32_t s_q[NW][WQ];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t *wq = s_q[wid];
    uint32_t qn = 0;   // warp-uniform count of staged appends
    unsigned long long nv = 0, ne = 0, nu = 0;
    bool chg = false, ovf = false;
    const uint32_t gw = (blockIdx.x * B + threadIdx.x) >> 5, nwarps = (gridDim.x * B) >> 5;
    const uint32_t wstride = nwarps * 32;

    auto wflush = [&](uint32_t thresh) {
        if (qn > thresh) {
            uint32_t b = 0;
            if (lane == 0) b = atomicAdd(&c->out_len, qn);
            b = __shfl_sync(FULL, b, 0);
            __syncwarp();
            for (uint32_t i = lane; i < qn; i += 32) out[b + i] = wq[i];
            __syncwarp();
            qn = 0;
        }
    };
    auto item_of = [&](uint32_t idx) -> uint32_t {
        return idx < nitems ? (implicit ? idx : ld_stream(in + idx, pf)) : 0xffffffffu;
    };
    // software pipeline: u1 = item of the current tile, u2 = item of the next
    // tile; pay1/beg1/end1 = value and row offsets of the current tile's item
    uint32_t wb = gw * 32;
    uint32_t u1 = item_of(wb + lane), u2 = item_of(wb + wstride + lane);
    uint32_t pay1 = 0, beg1 = 0, end1 = 0;
    if (u1 != 0xffffffffu) {
        if (ALGO != BFS) pay1 = (uint32_t)ld_val(a.val + u1, pl);
        beg1 = ld_ro(a.row_off + u1); end1 = ld_ro(a.row_off + u1 + 1);
    }

    for (; wb < nitems; wb += wstride) {   // warp-uniform
        const uint32_t u = u1, pay = pay1;
        uint32_t beg = beg1, deg = end1 - beg1;
        // issue the pipeline's next loads before touching this tile's arcs
        u1 = u2;
        u2 = item_of(wb + 2 * wstride + lane);
        if (u1 != 0xffffffffu) {
            if (ALGO != BFS) pay1 = (uint32_t)ld_val(a.val + u1, pl);
            beg1 = ld_ro(a.row_off + u1); end1 = ld_ro(a.row_off + u1 + 1);
        } else {
            pay1 = 0; beg1 = 0; end1 = 0;
        }
        if (u == 0xffffffffu || (ALGO == SSSP && pay == (uint32_t)INF)) deg = 0;
        else nv++;

        uint32_t incl = deg;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t total = __shfl_sync(FULL, incl, 31);
        const uint32_t excl = incl - deg;
        if (lane == 0) ne += total;

        for (uint32_t base = 0; base < total; base += 32 * U) {
            uint32_t e[U], v[U], p[U], uj[U];
            int32_t wt[U], cur[U];
            bool ok[U];
#pragma unroll
            for (int q = 0; q < U; q++) {
                const uint32_t k = base + q * 32 + lane;
                ok[q] = k < total;
                int j = 0;
#pragma unroll
                for (int st = 16; st > 0; st >>= 1) {
                    const uint32_t ex = __shfl_sync(FULL, excl, j + st);
                    if (ex <= k) j += st;
                }
                const uint32_t bj = __shfl_sync(FULL, beg, j), xj = __shfl_sync(FULL, excl, j);
                p[q] = __shfl_sync(FULL, pay, j);
                uj[q] = __shfl_sync(FULL, u, j);
                e[q] = bj + (k - xj);
            }
#pragma unroll
            for (int q = 0; q < U; q++) {
                v[q] = 0; wt[q] = 0;
                if (ok[q]) {
                    if (ALGO == SSSP) {   // one 8-byte (col, w) word: one DRAM burst per row
                        const uint2 x = ld_stream2(a.cw + e[q], pf);
                        v[q] = x.x; wt[q] = (int32_t)x.y;
                    } else {
                        v[q] = ld_stream(a.col + e[q], pf);
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < U; q++) {
                cur[q] = 0;
                if (ok[q]) {
                    if (ALGO == BFS) cur[q] = bit_test(a.vis, v[q]) ? 0 : INF;
                    else cur[q] = ld_val(a.val + v[q], pl);
                }
            }
            bool need[U];
            uint32_t citem[U];
#pragma unroll
            for (int q = 0; q < U; q++) {
                need[q] = false; citem[q] = 0;
                if (!ok[q]) continue;
                if (ALGO == SSSP) {
                    const uint32_t cand = p[q] + (uint32_t)wt[q];
                    if (cand >= (uint32_t)INF) {
                        ovf = true;
                    } else if ((int32_t)cand < cur[q]) {
                        atomicMin(a.val + v[q], (int32_t)cand);   // result unused: RED.MIN
                        nu++; chg = true; need[q] = true; citem[q] = v[q];
                    }
                } else if (ALGO == BFS) {
                    // t.dist > lev+1 -> t.dist = lev+1 (plain store;
                    // concurrent writers store the same value, R9)
                    if (cur[q] == INF) {
                        if (STYLE == WORKLIST) {   // the queue needs exactly-once: claim
                            need[q] = true; citem[q] = v[q];
                        } else {   // the level is written by the next round's k_scan
                            atomicOr(a.vis + (v[q] >> 5), 1u << (v[q] & 31));
                            atomicOr(bm_now + (v[q] >> 5), 1u << (v[q] & 31));
                            nu++; chg = true;
                        }
                    }
                } else {   // CC: hook the larger root under the smaller (min-label)
                    const uint32_t lu = p[q], lv = (uint32_t)cur[q];
                    if (lu != lv) {
                        const uint32_t hi = lu > lv ? lu : lv, lo = lu > lv ? lv : lu;
                        atomicMin(a.val + hi, (int32_t)lo);   // RED.MIN
                        nu++; chg = true;
                        if (STYLE == WORKLIST) { need[q] = true; citem[q] = uj[q]; }   // keep u while unresolved
                    }
                }
            }
            if (STYLE == VERTEX) {
                if (ALGO == SSSP) {
#pragma unroll
                    for (int q = 0; q < U; q++)
                        if (need[q]) atomicOr(bm_now + (citem[q] >> 5), 1u << (citem[q] & 31));
                }
            } else {
                uint32_t got[U];
#pragma unroll
                for (int q = 0; q < U; q++) {
                    got[q] = 0xffffffffu;
                    if (!need[q]) continue;
                    uint32_t *bmp = ALGO == BFS ? a.vis : bm_now;
                    got[q] = atomicOr(bmp + (citem[q] >> 5), 1u << (citem[q] & 31));
                }
#pragma unroll
                for (int q = 0; q < U; q++) {
                    const bool want = need[q] && !(got[q] & (1u << (citem[q] & 31)));
                    if (ALGO == BFS && want) { a.val[citem[q]] = (int32_t)(lev + 1); nu++; chg = true; }
                    const unsigned mask = __ballot_sync(FULL, want);
                    if (want) wq[qn + __popc(mask & ((1u << lane) - 1u))] = citem[q];
                    qn += __popc(mask);
                }
                __syncwarp();
                wflush(WQ > 32 * U ? WQ - 32 * U : 0);
            }
        }
    }
    if (STYLE == WORKLIST) { __syncwarp(); wflush(0); }
    flush_counters<B>(a, nv, ne, nu, chg, ovf, ALGO == BFS && STYLE == VERTEX);
}

// ------------------------------------------------------------------ EDGE style (COO)
// QP quads of four CSR-ordered arcs per thread per step: all QP 16-byte src
// loads are issued first and the sources' activity bits (bm[(r-1)%3],
// L1/L2-resident) tested, so a mostly-inactive round streams src[] with QP
// loads in flight per thread; col/w are fetched only for quads with an
// active source.
template <int ALGO>
__device__ __forceinline__ void edge_quad(const Args &a, uint32_t q, const uint32_t (&s)[4], uint32_t actmask,
                                          uint32_t m4, uint32_t tail, uint32_t lev, uint32_t *bm_now, uint64_t pf,
                                          uint64_t pl, unsigned long long &ne, unsigned long long &nu, bool &chg,
                                          bool &ovf) {
    uint32_t d[4] = {0, 0, 0, 0}, pay[4] = {0, 0, 0, 0};
    int32_t ww[4] = {0, 0, 0, 0};
    if (q < m4) {
        if (ALGO == SSSP) {
            const uint4 x0 = ld_stream4(a.cw + 4ull * q, pf), x1 = ld_stream4(a.cw + 4ull * q + 2, pf);
            d[0] = x0.x; ww[0] = (int32_t)x0.y; d[1] = x0.z; ww[1] = (int32_t)x0.w;
            d[2] = x1.x; ww[2] = (int32_t)x1.y; d[3] = x1.z; ww[3] = (int32_t)x1.w;
        } else {
            const uint4 d4 = ld_stream4(a.col + 4ull * q, pf);
            d[0] = d4.x; d[1] = d4.y; d[2] = d4.z; d[3] = d4.w;
        }
    } else {
        for (uint32_t j = 0; j < tail; j++) {
            if (ALGO == SSSP) {
                const uint2 x = ld_stream2(a.cw + 4ull * q + j, pf);
                d[j] = x.x; ww[j] = (int32_t)x.y;
            } else {
                d[j] = ld_stream(a.col + 4ull * q + j, pf);
            }
        }
    }
    int32_t cur[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
        cur[j] = 0;
        if (!((actmask >> j) & 1u)) continue;
        if (ALGO != BFS) pay[j] = (uint32_t)ld_val(a.val + s[j], pl);   // consecutive arcs share a source
        if (ALGO == BFS) cur[j] = bit_test(a.vis, d[j]) ? 0 : INF;
        else cur[j] = ld_val(a.val + d[j], pl);
    }
    // fire-and-forget relaxations (reductions), see k_expand_warp
#pragma unroll
    for (int j = 0; j < 4; j++) {
        if (!((actmask >> j) & 1u)) continue;
        ne++;
        if (ALGO == SSSP) {
            const uint32_t cand = pay[j] + (uint32_t)ww[j];
            if (cand >= (uint32_t)INF) { ovf = true; continue; }
            if ((int32_t)cand < cur[j]) {
                atomicMin(a.val + d[j], (int32_t)cand);
                atomicOr(bm_now + (d[j] >> 5), 1u << (d[j] & 31));
                nu++; chg = true;
            }
        } else if (ALGO == BFS) {   // e.src.dist == lev (R14) via the bitmap
            if (cur[j] == INF) {
                atomicOr(a.vis + (d[j] >> 5), 1u << (d[j] & 31));
                a.val[d[j]] = (int32_t)(lev + 1);
                atomicOr(bm_now + (d[j] >> 5), 1u << (d[j] & 31));
                nu++; chg = true;
            }
        } else {
            const uint32_t lu = pay[j], lv = (uint32_t)cur[j];
            if (lu != lv) {
                const uint32_t hi = lu > lv ? lu : lv, lo = lu > lv ? lv : lu;
                atomicMin(a.val + hi, (int32_t)lo);
                nu++; chg = true;
            }
        }
    }
}

template <int ALGO, int B, int QP>
__global__ void __launch_bounds__(B) k_edge(Args a) {
    Ctrl *c = a.ctrl;
    if (c->done) return;
    const uint32_t iter = c->iter, lev = iter - 1;
    clear_next_bitmap(a, iter);
    const uint32_t *bm_prev = bm_of(a, iter - 1);
    uint32_t *bm_now = bm_of(a, iter);
    const uint64_t pf = pol_evict_first(), pl = pol_evict_last();
    const uint32_t m4 = a.m >> 2, tail = a.m & 3u;
    const uint32_t nq = m4 + (tail ? 1u : 0u);
    unsigned long long ne = 0, nu = 0;
    bool chg = false, ovf = false;
    const uint32_t stride = gridDim.x * B;
    for (uint32_t q0 = blockIdx.x * B + threadIdx.x; q0 < nq; q0 += stride * QP) {
        uint32_t s[QP][4];
        uint32_t act[QP];
#pragma unroll
        for (int p = 0; p < QP; p++) {
            const uint32_t q = q0 + p * stride;
            s[p][0] = s[p][1] = s[p][2] = s[p][3] = 0;
            if (q < m4) {
                const uint4 s4 = ld_stream4(a.src + 4ull * q, pf);
                s[p][0] = s4.x; s[p][1] = s4.y; s[p][2] = s4.z; s[p][3] = s4.w;
            } else if (q < nq) {
                for (uint32_t j = 0; j < tail; j++) s[p][j] = ld_stream(a.src + 4ull * q + j, pf);
            }
        }
#pragma unroll
        for (int p = 0; p < QP; p++) {
            const uint32_t q = q0 + p * stride;
            const uint32_t cntq = q < m4 ? 4u : (q < nq ? tail : 0u);
            act[p] = 0;
#pragma unroll
            for (int j = 0; j < 4; j++)   // ALGO == CC: every arc hooks; otherwise the source must be active
                if ((uint32_t)j < cntq && (ALGO == CC || bit_test(bm_prev, s[p][j]))) act[p] |= 1u << j;
        }
#pragma unroll
        for (int p = 0; p < QP; p++)
            if (act[p]) edge_quad<ALGO>(a, q0 + p * stride, s[p], act[p], m4, tail, lev, bm_now, pf, pl, ne, nu, chg, ovf);
    }
    flush_counters<B>(a, 0ull, ne, nu, chg, ovf);
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
template <int ALGO, int STYLE>
__global__ void k_advance(Ctrl *c, cudaGraphConditionalHandle h, int in_graph, uint32_t launches_per_round,
                          uint32_t n, uint32_t pull_div) {
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
        } else if (STYLE == VERTEX) {
            c->in_len = 0;   // k_scan rebuilds the frontier of the next round
            // direction-optimising BFS: bottom-up while the next frontier is large
            if (ALGO == BFS) c->pull = pull_div && c->found > n / pull_div;
        }
        c->found = 0;
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

__global__ void k_interleave(uint64_t m, const uint32_t *col, const int32_t *w, uint2 *cw) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride)
        cw[e] = make_uint2(col[e], (uint32_t)w[e]);
}

// Reverse CSR (in-arcs), built on the device: in-degree histogram, scan,
// scatter (in-row order is arbitrary: BFS levels do not depend on it).
__global__ void k_indeg(uint64_t m, const uint32_t *col, uint32_t *cnt) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) atomicAdd(cnt + col[e], 1u);
}
// exclusive scan of x[0..len) in place, tiles of 1024 (two-level, second
// level over tile sums done by k_scan_tiles with one CTA)
__global__ void k_scan_local(uint32_t *x, uint64_t len, uint32_t *tile_sums) {
    __shared__ uint32_t s_warp[32];
    const uint64_t i0 = (uint64_t)blockIdx.x * 1024 + threadIdx.x * 4;
    uint32_t v[4], sum = 0;
    for (int j = 0; j < 4; j++) { v[j] = i0 + j < len ? x[i0 + j] : 0; sum += v[j]; }
    uint32_t total;
    uint32_t run = block_excl_scan<256>(sum, total, s_warp);
    for (int j = 0; j < 4; j++) { if (i0 + j < len) x[i0 + j] = run; run += v[j]; }
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}
__global__ void k_scan_tiles(uint32_t *tile_sums, uint32_t ntiles) {
    __shared__ uint32_t s_warp[32];
    uint32_t carry = 0;
    for (uint32_t b0 = 0; b0 < ntiles; b0 += 1024) {
        const uint32_t i0 = b0 + threadIdx.x * 4;
        uint32_t v[4], sum = 0;
        for (int j = 0; j < 4; j++) { v[j] = i0 + j < ntiles ? tile_sums[i0 + j] : 0; sum += v[j]; }
        uint32_t total;
        uint32_t run = block_excl_scan<256>(sum, total, s_warp) + carry;
        for (int j = 0; j < 4; j++) { if (i0 + j < ntiles) tile_sums[i0 + j] = run; run += v[j]; }
        carry += total;
    }
}
__global__ void k_scan_add(uint32_t *x, uint64_t len, const uint32_t *tile_sums) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < len) x[i] += tile_sums[i / 1024];
}
__global__ void k_rev_scatter(uint32_t n, const uint32_t *row_off, const uint32_t *col, uint32_t *cursor,
                              uint32_t *rin_col) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += stride)
        for (uint32_t e = row_off[u]; e < row_off[u + 1]; e++) rin_col[atomicAdd(cursor + col[e], 1u)] = u;
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
