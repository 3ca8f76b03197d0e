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
#ifdef FK_PROBE
__device__ int fk_probe_mode;   // tools/expand_probe.cu only (never defined in the product build)
#endif
constexpr unsigned FULL = 0xffffffffu;
constexpr uint32_t NONE = 0xffffffffu;   // "no item / no vertex"

enum Algo : int { SSSP = 0, BFS = 1, CC = 2 };
enum Style : int { VERTEX = 0, EDGE = 1, WORKLIST = 2, DELTA = 3,
                   VFUSED = 4 /* partitioned VERTEX rounds writing remote targets into their owners (partition.cuh) */ };
__host__ __device__ constexpr bool is_vertex(int style) { return style == VERTEX || style == VFUSED; }
enum DeltaMode : uint32_t { MODE_NEAR = 0, MODE_SCAN = 1 };
enum DevStatus : int { ST_OK = 0, ST_OVERFLOW = 5, ST_NOT_CONVERGED = 6, ST_QUEUE = 7 /* internal: queue bound */ };

// Device-resident control block: the convergence decision lives here, so no
// host round trip happens per round (replaces the per-iteration `changed`
// copy of PAPER.md:1682-1684 / SPEC.md:370).
struct Ctrl {
    uint32_t iter;        // current round, 1-based
    uint32_t in_len;      // items in the input frontier (queue styles)
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
    uint32_t visited;     // BFS: vertices discovered so far (direction heuristic)
    unsigned long long rnd_items, rnd_edges;   // BFS VERTEX: items expanded / arcs scanned this round
    uint32_t lazy;        // BFS VERTEX: this push round marks discoveries in the round bitmap only
    uint32_t merge;       // BFS VERTEX: last round was lazy -- its discoveries are not in vis yet
    uint32_t lazy_found;  // BFS VERTEX: `found` of the last lazy round (counts a vertex once per marking arc)
    uint32_t exact;       // BFS VERTEX: its discoveries counted exactly while they are merged into vis
    uint32_t thr;         // DELTA: current bucket threshold T (near: dist < T)
    uint32_t delta;       // DELTA: bucket width
    uint32_t minpend;     // DELTA: min tentative distance parked in the far set
    uint32_t delta0;      // DELTA: initial bucket width (adaptive mode never goes below it)
    uint32_t delta_adapt; // DELTA: adapt the bucket width per bucket (auto Δ)
    uint32_t bk_rounds;   // DELTA: near rounds of the current bucket
    uint32_t delta_cap;   // DELTA: adaptive growth cap, in multiples of delta0
    unsigned long long bk_items;   // DELTA: items relaxed in the current bucket's near rounds
    uint32_t mode;        // DELTA: MODE_NEAR (relax the near queue) / MODE_SCAN (refill from far)
    uint32_t bar_arrive;  // persistent kernel: CTAs arrived at the grid barrier
    uint32_t bar_gen;     // persistent kernel: barrier generation
    uint32_t blk;         // this round expands over the destination-blocked layout (dense rounds)
    uint32_t noq;         // WORKLIST: this (dense) round marks the bitmap only -- no queue is built
    uint32_t prevnoq;     // WORKLIST / DELTA: the previous round did: read this round's items from the bitmap
    uint32_t hooks;       // MST: components hooked this round
    uint32_t cand_ovf;    // SSSP: some candidate d[u]+w reached INF (k_overflow_check decides, reading R3)
    unsigned long long wsum;       // MST: total weight of the forest edges chosen so far
    unsigned long long xremote;    // fused partitioned rounds: improvements sent to other parts (RED pairs)
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
    // destination-blocked layout (SSSP): the arcs of block k
    // (targets in [k*bsz, (k+1)*bsz)) form their own CSR; rowb[k*(n+1)+u] is
    // the first arc of row u in block k.  nblk == 1: rowb/cwb/srcb alias
    // row_off/cw/src.
    const uint32_t *rowb;      // [nblk*(n+1)]
    const uint2 *cwb;          // [m]
    const uint32_t *srcb;      // [m] EDGE style
    const uint2 *chunk;        // source range [min, max] of each EDGE chunk of src (CSR order; BFS chunk size)
    const uint2 *chunkb;       // ... of srcb (blocked order) or src, in SSSP chunks
    uint32_t nblk;
    uint32_t dense_div;        // a round is dense when its frontier exceeds n / dense_div (0: never)
    uint32_t blk_div;          // ... and walks the blocked layout when it exceeds n / blk_div (0: never)
    uint32_t wl_noq;           // WORKLIST dense rounds mark like VERTEX (no claim / queue); 0 = off
    uint32_t dl_noq;           // ... DELTA dense rounds (near marks in the bitmap, far parking as usual)
    uint32_t cta_thr;          // rows longer than this are expanded by the whole CTA (0: warp-level only)
    uint32_t wl_pull;          // BFS WORKLIST: rounds may run bottom-up (k_pull) like VERTEX (0: push only)
    uint32_t skip_now;         // SSSP: an item whose bit is already set in this round's bitmap (improved again
                               // this round, so expanded next round with its newer value) is not expanded now
    uint32_t lazy_div;         // BFS VERTEX: a push round whose frontier exceeds n / lazy_div marks only the
                               // round bitmap; the next round's k_pull merges it into vis (0: never)
    // fused partitioned rounds (VFUSED): owned range, part bounds and the
    // owners' value arrays / round bitmaps (peer memory on real GPUs)
    uint32_t lo, hi, nparts;
    const uint32_t *bounds;
    int32_t *const *peer_val;
    uint32_t *const *peer_bm;
    uint32_t delta_adapt;      // DELTA: adapt the bucket width per bucket (auto Δ)
    uint32_t delta_cap;        // ... up to delta_cap x the initial width (0: 128)
    uint32_t local_tiles;      // SSSP DELTA sparse rounds: local continuation tiles per warp (0 = off)
    uint32_t local_max;        // ... in rounds of at most local_max items
    uint32_t wl_local_tiles;   // the same for SSSP WORKLIST sparse rounds
    uint32_t wl_local_max;
    const uint32_t *rin_off;   // [n+1] reverse CSR (in-arcs), BFS pull only
    const uint32_t *rin_col;   // [m]
    int32_t *val;              // dist / level / label [n]
    uint8_t *lv8;              // BFS: levels < 255 as bytes [n] (0xFF: none), merged into val by k_bfs_levels
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
#ifdef FK_NO_EVICT_FIRST
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
#else
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
#endif
    return p;
}
__device__ __forceinline__ uint64_t pol_evict_last() {
    uint64_t p;
#ifdef FK_NO_EVICT_LAST
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
#else
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
#endif
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

// Frontier-queue append (fr0 / fr1 hold n + 1 entries).  Claims make every
// round's appends distinct, so the bound is never reached; an append past it
// is dropped and flagged (ST_QUEUE: the call fails with FALCON_ERR_CUDA and
// no kernel writes outside the queue).
__device__ __forceinline__ void q_put(const Args &a, uint32_t *out, uint32_t idx, uint32_t v) {
    if (idx <= a.n) out[idx] = v;
    else a.ctrl->status = ST_QUEUE;
}

// BFS level L of vertex v (PAPER.md:1309 `t.dist = lev+1`).  Levels below 255
// go to a byte array (n bytes: L2-resident at 25M vertices, where the int32
// array is 100 MB): each round's scattered level stores would otherwise
// partially dirty most sectors of the 100 MB value array and cost a DRAM
// read-modify-write of all of it (ncu: ~200 MB per pull round on rand-25M).
// Deeper levels are stored in val directly; k_bfs_levels merges at the end.
__device__ __forceinline__ void put_level(const Args &a, uint32_t v, uint32_t L) {
    if (L < 255u) a.lv8[v] = (uint8_t)L;
    else a.val[v] = (int32_t)L;
}

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
    __syncwarp();      // bar.sync is .aligned: the warp must arrive converged (compute-sanitizer synccheck)
    __syncthreads();
    if (lane == 0) { s_red[0][wid] = nv; s_red[1][wid] = ne; s_red[2][wid] = nu; }
    if (chg) atomicOr(&s_flags, 1);
    if (ovf) atomicOr(&s_flags, 2);
    __syncwarp();
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t0 = 0, t1 = 0, t2 = 0;
        for (int i = 0; i < B / 32; i++) { t0 += s_red[0][i]; t1 += s_red[1][i]; t2 += s_red[2][i]; }
        unsigned long long *c = a.cnt + 3ull * blockIdx.x;   // this CTA's private slot: no atomics
        c[0] += t0; c[1] += t1; c[2] += t2;
        if (t2) atomicAdd(&a.ctrl->found, (uint32_t)(t2 < 0xffffffffull ? t2 : 0xffffffffull));   // density heuristics
        if (t0) atomicAdd(&a.ctrl->rnd_items, t0);   // direction heuristic (BFS VERTEX)
        if (t1) atomicAdd(&a.ctrl->rnd_edges, t1);
        if (s_flags & 1) a.ctrl->changed = 1;
        if (s_flags & 2) a.ctrl->cand_ovf = 1;   // not an error by itself (R3): checked after the fixpoint
    }
}

// Clear the bitmap of round r+1 (grid-stride, 16-byte stores).
__device__ __forceinline__ void clear_next_bitmap(const Args &a, uint32_t r) {
    uint4 *p = reinterpret_cast<uint4 *>(bm_of(a, r + 1));
    const uint32_t n4 = a.nwords >> 2;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x)
        p[i] = make_uint4(0, 0, 0, 0);
}

// ------------------------------------------------------------------ init (fused)
// SSSP/BFS: dist = MAX_INT, dist[source] = 0;
// CC: label[v] = v.  Clears the bitmaps (source bit set in bm0 / vis), seeds
// the frontier and resets the control block, in one launch.
template <int ALGO>
__global__ void k_init(Args a, uint32_t source, uint32_t cap, uint32_t cnt_len, int style, uint32_t delta) {
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t t0 = blockIdx.x * blockDim.x + threadIdx.x;
    if (ALGO == BFS) {   // levels start in the byte array (0xFF: none); val is written by k_bfs_levels
        uint4 *l4 = reinterpret_cast<uint4 *>(a.lv8);
        const uint32_t n16 = (a.n + 15) / 16;
        for (uint32_t i = t0; i < n16; i += stride) {
            uint4 x = make_uint4(~0u, ~0u, ~0u, ~0u);
            if (i == source / 16) {   // the source is at level 0
                const uint32_t keep = ~(0xFFu << (8 * (source % 4)));
                switch ((source % 16) / 4) {
                case 0: x.x &= keep; break;
                case 1: x.y &= keep; break;
                case 2: x.z &= keep; break;
                default: x.w &= keep; break;
                }
            }
            l4[i] = x;
        }
    } else {
        for (uint32_t v = t0; v < a.n; v += stride) {
            if (ALGO == CC) a.val[v] = (int32_t)v;
            else a.val[v] = v == source ? 0 : INF;
        }
    }
    const uint32_t sw = ALGO == CC ? 0xffffffffu : source >> 5, sb = 1u << (source & 31);
    for (uint32_t i = t0; i < a.nwords; i += stride) {
        a.bm0[i] = i == sw ? sb : 0u;
        a.bm1[i] = 0u; a.bm2[i] = 0u;
        if (ALGO == BFS) a.vis[i] = i == sw ? sb : 0u;
        else if (style == DELTA) a.vis[i] = 0u;   // the far set
    }
    for (uint32_t i = t0; i < cnt_len; i += stride) a.cnt[i] = 0ull;
    if (t0 == 0) {
        Ctrl *c = a.ctrl;
        c->iter = 1;
        c->in_len = ALGO == CC ? a.n : (style == VERTEX ? 0u : 1u);   // VERTEX: read from the bitmap
        c->out_len = 0; c->changed = 0; c->cap = cap; c->sel = 0; c->done = 0;
        c->all_active = ALGO == CC ? 1u : 0u;
        c->status = ST_OK; c->source = source;
        c->launches = 1; c->vertices = 0; c->edges = 0; c->updates = 0;
        c->pull = 0; c->found = 0; c->visited = 1; c->rnd_items = 0; c->rnd_edges = 0; c->lazy = 0; c->merge = 0; c->lazy_found = 0; c->exact = 0;
        c->thr = delta; c->delta = delta; c->minpend = 0xffffffffu; c->mode = MODE_NEAR;
        c->delta0 = delta; c->delta_adapt = a.delta_adapt; c->bk_rounds = 0; c->bk_items = 0;
        c->delta_cap = a.delta_cap ? a.delta_cap : 128u;
        c->bar_arrive = 0; c->blk = 0; c->noq = 0; c->prevnoq = 0; c->hooks = 0; c->wsum = 0; c->cand_ovf = 0;
        c->xremote = 0;
        if (ALGO != CC) a.fr0[0] = source;
    }
}

// BFS epilogue: val[v] = byte level if v got one, INF if v was never
// discovered; a vertex discovered at level >= 255 already has its level in
// val (put_level).  Four vertices per thread, a full 16-byte store when none
// of the four keeps its value -- val is never read for a shallow BFS.
__global__ void k_bfs_levels(Args a) {
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t n4 = (a.n + 3) / 4;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        const uint32_t b4 = reinterpret_cast<const uint32_t *>(a.lv8)[i];
        const uint32_t vw = (a.vis[i >> 3] >> ((i & 7) * 4)) & 0xFu;   // visited bits of vertices 4i .. 4i+3
        int32_t o[4];
        bool keep = false;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const uint32_t b = (b4 >> (8 * j)) & 0xFFu;
            const bool visited = (vw >> j) & 1u;
            o[j] = b != 0xFFu ? (int32_t)b : INF;
            if (b == 0xFFu && visited) keep = true;   // level >= 255, in val already
        }
        if (!keep && 4 * i + 4 <= a.n) {
            reinterpret_cast<int4 *>(a.val)[i] = make_int4(o[0], o[1], o[2], o[3]);
        } else {
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const uint32_t v = 4 * i + j;
                const bool visited = (vw >> j) & 1u;
                if (v < a.n && !(((b4 >> (8 * j)) & 0xFFu) == 0xFFu && visited)) a.val[v] = o[j];
            }
        }
    }
}

// ------------------------------------------------------------------ DELTA: refill from the far set
// Δ-stepping (PAPER.md:454 / SPEC.md:415-418, 453-461)
// as a near/far worklist: the near queue holds vertices below the bucket
// threshold T, improved vertices at or beyond T are parked in the far set
// (a bitmap).  When the near queue runs dry, k_advance moves T to the bucket
// of the smallest parked distance and this pass (run by k_expand_warp in a
// scan round) moves every parked vertex
// now below T into the near queue (one warp per 32-vertex word: the far word
// is rewritten with a plain store), recomputing the minimum of what stays.
template <bool COHERENT>
__device__ __forceinline__ void scan_far_round(const Args &a, Ctrl *c, uint32_t iter, uint32_t thr, uint32_t *out,
                                               unsigned long long &nv) {
    // lane-per-word (coalesced 128-byte loads of the far bitmap); a lane walks
    // the set bits of its own word, then the warp compacts its moves
    uint32_t *bm_now = bm_of(a, iter);
    const int lane = threadIdx.x & 31;
    const uint32_t gt = blockIdx.x * blockDim.x + threadIdx.x, nthreads = gridDim.x * blockDim.x;
    uint32_t pend_min = 0xffffffffu;
    for (uint32_t w0 = gt - lane; w0 < a.nwords; w0 += nthreads) {   // warp-uniform
        const uint32_t wi = w0 + lane;
        const uint32_t fw = wi < a.nwords ? (COHERENT ? __ldcg(a.vis + wi) : a.vis[wi]) : 0u;
        uint32_t mv = 0;
        for (uint32_t x = fw; x; x &= x - 1) {
            const uint32_t v = wi * 32u + (uint32_t)(__ffs(x) - 1);
            const uint32_t d = (uint32_t)(COHERENT ? __ldcg(a.val + v) : a.val[v]);
            if (d < thr) mv |= x & (0u - x);
            else pend_min = d < pend_min ? d : pend_min;
        }
        const uint32_t cnt = __popc(mv);
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t total = __shfl_sync(FULL, incl, 31);
        if (total == 0) continue;
        uint32_t b = 0;
        if (lane == 0) b = atomicAdd(&c->out_len, total);
        b = __shfl_sync(FULL, b, 0) + incl - cnt;
        if (mv) {
            a.vis[wi] = fw & ~mv;
            atomicOr(bm_now + wi, mv);   // these are the near queue of the next round
            for (uint32_t x = mv; x; x &= x - 1) q_put(a, out, b++, wi * 32u + (uint32_t)(__ffs(x) - 1));
        }
        nv += cnt;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint32_t y = __shfl_xor_sync(FULL, pend_min, o);
        pend_min = y < pend_min ? y : pend_min;
    }
    if (lane == 0 && pend_min != 0xffffffffu) atomicMin(&c->minpend, pend_min);
}

// Sum of the arc weights (auto Δ = max(1, average weight)).
__global__ void k_sum_weights(uint64_t m, const int32_t *w, unsigned long long *sum) {
    unsigned long long t = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) t += (uint32_t)w[e];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(FULL, t, o);
    if ((threadIdx.x & 31) == 0 && t) atomicAdd(sum, t);
}

// ------------------------------------------------------------------ BFS bottom-up (pull) round
// Direction-optimising BFS, VERTEX style over `innbrs` (Table
// "Iterators"): every unvisited vertex scans its in-arcs until it finds a
// parent in the previous level (bm[(r-1)%3]).  Run when the frontier is large
// (k_advance).
//
// Two forms, chosen per round by bfs_direction (Ctrl::pull):
//  1 = word: a warp owns one bitmap word at a time, lane i scans the in-arcs
//      of vertex 32w + i if it is unvisited -- for a large unvisited set,
//      where most lanes have work;
//  2 = compacted: a warp owns groups of PG = 16 words (512 vertices, one word
//      per lane); the group's UNVISITED vertices are compacted into a
//      shared-memory list and walked two per lane, so every lane carries two
//      independent early-exit scans (rin_col load -> parent bit test) however
//      few vertices of a word are still unvisited (the word form left most
//      lanes idle when 6 % of the vertices were unvisited: rand-25M 150 us
//      -> 95 us for that round, but 309 -> 370 us on a round with 72 %).
//      Parents found are collected in a per-warp shared word array, so the
//      visited / next-frontier words are written once, with plain stores, by
//      the lane owning the word.
template <int B>
__global__ void __launch_bounds__(B, 2048 / B) k_pull(Args a) {   // 8 CTAs of 256 per SM: 32 registers
    Ctrl *c = a.ctrl;
    if (c->done) return;
    if (!c->pull) {
        // lazy visited set (Ctrl::lazy): a heavy push round sets only the
        // round bitmap; the vertices it discovered join the visited bitmap
        // here, before the next round's expansion tests it
        if (c->merge) {
            const uint4 *p4 = reinterpret_cast<const uint4 *>(bm_of(a, c->iter - 1));
            uint4 *v4 = reinterpret_cast<uint4 *>(a.vis);
            uint32_t fresh = 0;
            for (uint32_t i = blockIdx.x * B + threadIdx.x; i < a.nwords / 4; i += gridDim.x * B) {
                const uint4 p = p4[i];
                if (p.x | p.y | p.z | p.w) {
                    uint4 v = v4[i];
                    fresh += __popc(p.x & ~v.x) + __popc(p.y & ~v.y) + __popc(p.z & ~v.z) + __popc(p.w & ~v.w);
                    v.x |= p.x; v.y |= p.y; v.z |= p.z; v.w |= p.w;
                    v4[i] = v;
                }
            }
            fresh = __reduce_add_sync(FULL, fresh);
            if ((threadIdx.x & 31) == 0 && fresh) atomicAdd(&c->exact, fresh);
        }
        return;
    }
    const uint32_t iter = c->iter, lev = iter - 1;
    clear_next_bitmap(a, iter);
    if (blockIdx.x == 0 && threadIdx.x == 0) c->noq = 1;   // WORKLIST: the next round reads its items from bm_now
    const uint32_t *bm_prev = bm_of(a, iter - 1);
    uint32_t *bm_now = bm_of(a, iter);
    const bool merge = c->merge != 0;   // (vis lacks last round's discoveries: visw |= prevw below, written back)
    if (c->pull == 1) {
        const int lane = threadIdx.x & 31;
        uint32_t fresh = 0;   // last (lazy) round's discoveries, counted once each
        const uint32_t gw = (blockIdx.x * B + threadIdx.x) >> 5, nwarps = (gridDim.x * B) >> 5;
        uint32_t nv = 0, ne = 0, nu = 0;   // per-thread counts (32-bit: registers)
        bool chg = false;
        for (uint32_t wi = gw; wi < a.nwords; wi += nwarps) {
            const uint32_t prevw = bm_prev[wi];
            const uint32_t vis0 = a.vis[wi];
            const uint32_t visw = vis0 | prevw;   // (a lazy visited set lacks last round's discoveries)
            if (merge && lane == 0) fresh += __popc(prevw & ~vis0);
            const uint32_t v = wi * 32u + lane;
            if ((prevw >> lane) & 1u) put_level(a, v, lev);   // discovered last round
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
            if (lane == 0) {
                if (mask || (merge && prevw)) a.vis[wi] = visw | mask;
                if (mask) bm_now[wi] = mask;
            }
            if (found) { nu++; chg = true; }
        }
        if (merge) {
            fresh = __reduce_add_sync(FULL, fresh);
            if ((threadIdx.x & 31) == 0 && fresh) atomicAdd(&c->exact, fresh);
        }
        flush_counters<B>(a, nv, ne, nu, chg, false);
        return;
    }
    // 16-word groups: 16.5 KB of shared memory per CTA keeps 8 CTAs of 256
    // threads resident per SM (one wave), and a round has enough groups per
    // warp to balance (32-word groups: 6 CTAs/SM, two waves, 2x slower)
    constexpr uint32_t PG = 16;
    __shared__ uint32_t s_it[B / 32][PG * 32];
    __shared__ uint32_t s_fd[B / 32][PG];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t *sit = s_it[wid], *sfd = s_fd[wid];
    const uint32_t gw = (blockIdx.x * B + threadIdx.x) >> 5, nwarps = (gridDim.x * B) >> 5;
    uint32_t nv = 0, ne = 0, nu = 0;   // per-thread counts (32-bit: registers)
    bool chg = false;
    uint32_t fresh = 0;
    for (uint32_t g0 = gw * PG; g0 < a.nwords; g0 += nwarps * PG) {   // warp-uniform
        const uint32_t wi = g0 + lane;
        uint32_t visw = 0xffffffffu, prevw = 0;
        if (lane < PG && wi < a.nwords) {
            prevw = bm_prev[wi];
            const uint32_t vis0 = a.vis[wi];
            visw = vis0 | prevw;
            if (merge) fresh += __popc(prevw & ~vis0);
        }
        // the level of the vertices discovered last round: one coalesced
        // 128-byte store per non-empty word
        for (unsigned pm = __ballot_sync(FULL, prevw != 0); pm; pm &= pm - 1) {   // warp-uniform
            const int j = __ffs(pm) - 1;
            if ((__shfl_sync(FULL, prevw, j) >> lane) & 1u) put_level(a, (g0 + j) * 32u + lane, lev);
        }
        uint32_t unv = ~visw;
        const uint64_t v0w = (uint64_t)wi * 32u;   // vertices >= n count as visited
        if (v0w >= a.n) unv = 0;
        else if (v0w + 32 > a.n) unv &= (1u << (uint32_t)(a.n - v0w)) - 1u;
        const uint32_t cnt = __popc(unv);
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t total = __shfl_sync(FULL, incl, 31);
        if (total == 0) continue;
        uint32_t pos = incl - cnt;
        for (uint32_t y = unv; y; y &= y - 1) sit[pos++] = wi * 32u + (uint32_t)(__ffs(y) - 1);
        if (lane < PG) sfd[lane] = 0u;
        __syncwarp();
        nv += cnt;
        for (uint32_t j0 = 0; j0 < total; j0 += 64) {   // warp-uniform
            const uint32_t va = j0 + lane < total ? sit[j0 + lane] : NONE;
            const uint32_t vb = j0 + 32 + lane < total ? sit[j0 + 32 + lane] : NONE;
            uint32_t ea = 0, eae = 0, eb = 0, ebe = 0;
            if (va != NONE) { ea = ld_ro(a.rin_off + va); eae = ld_ro(a.rin_off + va + 1); }
            if (vb != NONE) { eb = ld_ro(a.rin_off + vb); ebe = ld_ro(a.rin_off + vb + 1); }
            bool fa = false, fb = false;
            while (ea < eae || eb < ebe) {   // two independent early-exit scans per lane
                const bool la = ea < eae, lb = eb < ebe;
                const uint32_t sa = la ? ld_ro(a.rin_col + ea) : 0u;
                const uint32_t sb = lb ? ld_ro(a.rin_col + eb) : 0u;
                const bool ha = la && bit_test(bm_prev, sa);
                const bool hb = lb && bit_test(bm_prev, sb);
                ne += (uint32_t)la + (uint32_t)lb;
                if (ha) { fa = true; ea = eae; } else ea += la;
                if (hb) { fb = true; eb = ebe; } else eb += lb;
            }
            if (fa) atomicOr(sfd + ((va >> 5) - g0), 1u << (va & 31));
            if (fb) atomicOr(sfd + ((vb >> 5) - g0), 1u << (vb & 31));
        }
        __syncwarp();
        const uint32_t nw = lane < PG ? sfd[lane] : 0u;
        if (merge && prevw && !nw && lane < PG) a.vis[wi] = visw;   // last round's discoveries join
        if (nw) {
            a.vis[wi] = visw | nw;
            bm_now[wi] = nw;
            nu += __popc(nw);
            chg = true;
        }
        __syncwarp();
    }
    if (merge) {
        fresh = __reduce_add_sync(FULL, fresh);
        if ((threadIdx.x & 31) == 0 && fresh) atomicAdd(&c->exact, fresh);
    }
    flush_counters<B>(a, nv, ne, nu, chg, false);
}

// ------------------------------------------------------------------ warp-centric expansion
// A WARP owns 32 items (frontier entries or active vertices): a shuffle scan
// turns their out-degrees into offsets and the warp walks the concatenated
// arc ranges 32*U arcs at a time, each lane finding its item by a 5-step
// shuffle binary search -- every arc gets one lane whatever the degree
// distribution (cooperative expansion for skewed RMAT degrees, PAPER.md:
// 441-446) and consecutive lanes read consecutive arc words.  There is no
// block barrier in the loop.
//
// Where the items come from:
//  * sparse rounds (queue styles, small frontier): the frontier queue,
//    item loads software-pipelined two tiles ahead;
//  * dense rounds (VERTEX always; queue styles when the frontier exceeds
//    n / dense_div): the activity bitmap of the previous round, 32 words
//    (1024 vertices) per warp step, compacted in shared memory -- items come
//    out in vertex order, so row offsets and arcs are read as ascending
//    streams instead of one random row per item.
//
// Destination blocking (SSSP dense rounds): the value array
// of a 25M-vertex graph (100 MB) does not stay in L2 next to the streamed
// arcs, and every gather that misses costs a DRAM sector.  The arcs are
// therefore stored a second time split by target block (nblk blocks of bsz
// vertices, bsz*4 bytes sized to stay L2-resident); a dense round walks the
// frontier once per block, so at any time all warps gather from one block.
//
// Relaxations:
//  * VERTEX: fire-and-forget -- the read filter `cand < val[v]` decides,
//    atomicMin / the bitmap OR are issued as reductions (RED) whose results
//    nobody waits for.  A vertex whose read passed the filter is improved in
//    this round -- by us, or by whoever lowered it further after our read,
//    who marks it too -- so the marked set is exactly the set of vertices
//    improved this round (R8);
//  * queue styles (WORKLIST, DELTA) need the old bitmap word to append each
//    vertex once; the bitmap bits of the items being expanded are cleared on
//    the way (every set bit of bm[(r-1)%3] is an item of round r), so the
//    bitmap is clean again when it is reused two rounds later.
struct RoundAcc {
    unsigned long long nv = 0, ne = 0, nu = 0;
    bool chg = false, ovf = false;
};

// COHERENT: loads of data written earlier in the same (persistent) kernel
// bypass L1 (ld.global.cg); otherwise the read-only / evict-first paths.
template <bool COHERENT>
__device__ __forceinline__ uint32_t ld_item(const uint32_t *p, uint64_t pf) {
    if (COHERENT) return __ldcg(p);
    return ld_stream(p, pf);
}
template <bool COHERENT>
__device__ __forceinline__ int32_t ld_value(const int32_t *p, uint64_t pl) {
    if (COHERENT) return __ldcg(p);
    return ld_val(p, pl);
}

// Per-round, per-warp expansion state.
struct Xw {
    const uint32_t *rows;   // row offsets of the current block (or the plain CSR)
    const uint2 *arcs;      // (col, w) words (SSSP)
    uint32_t *bm_now, *bm_prev, *out, *wq;
    Ctrl *c;
    uint32_t lev, thr, qh, qn, pend_min;   // wq[qh, qn): staged appends / the local stack (LOCAL)
    uint64_t pf, pl;
    // CTA-level expansion: rows longer than hthr arcs are handed to the CTA
    // (shared list hb/hd/hp of HMAX rows, count *hn; hthr = 0: off)
    uint32_t *hb, *hd, *hp, *hn;
    uint32_t hthr;
    bool lazy;   // BFS VERTEX lazy push round (Ctrl::lazy)
};
constexpr uint32_t HMAX = 64;   // long rows per CTA and round (more: the warp expands them itself)

// Local continuation (LOCAL rounds): hand the warp's unexpanded local items
// wq[qh, qn) over to the next round -- claim each in this round's bitmap and
// append the newly claimed ones to the queue.
__device__ __forceinline__ void spill_local(const Args &a, Xw &x) {
    const int lane = threadIdx.x & 31;
    for (uint32_t i0 = x.qh; i0 < x.qn; i0 += 32) {   // warp-uniform
        const uint32_t i = i0 + lane;
        uint32_t v = 0;
        bool want = false;
        if (i < x.qn) {
            v = x.wq[i];
            want = !(atomicOr(x.bm_now + (v >> 5), 1u << (v & 31)) & (1u << (v & 31)));
        }
        const unsigned mask = __ballot_sync(FULL, want);
        if (!mask) continue;
        uint32_t b = 0;
        if (lane == 0) b = atomicAdd(&x.c->out_len, (uint32_t)__popc(mask));
        b = __shfl_sync(FULL, b, 0);
        if (want) q_put(a, x.out, b + __popc(mask & ((1u << lane) - 1u)), v);
    }
    __syncwarp();
    x.qh = x.qn = 0;
}

template <int ALGO, bool COHERENT>
__device__ __forceinline__ void item_rows(const Args &a, const Xw &x, uint32_t u, uint32_t &pay, uint32_t &beg,
                                          uint32_t &end) {
    pay = 0; beg = 0; end = 0;
    if (u != NONE) {   // the item's own value and offsets: streamed, evict-first (keep L2 for the gathers)
        if (ALGO != BFS) pay = (uint32_t)ld_value<COHERENT>(a.val + u, x.pf);
        beg = ld_stream(x.rows + u, x.pf); end = ld_stream(x.rows + u + 1, x.pf);
    }
}

// One step of 32*U arcs whose (col, w) loads have been issued; relaxed one
// step later (cross-tile software pipeline, see relax_tile).
template <int U>
struct Step {
    uint32_t v[U], p[U];
    int32_t wt[U];
    bool ok[U];
    bool live;
};

// Gather the targets' values of a loaded step and relax its arcs.  NOQ: a
// dense WORKLIST round marks improved vertices like VERTEX does (reductions,
// no claim, no queue append): its successor reads the frontier from the bitmap.
// LOCAL: an improved in-bucket target is pushed unclaimed onto the warp's
// local stack wq[qh, qn) (FIFO), which the warp expands itself later in the
// round (expand_round); what it leaves over is claimed and queued then.
template <int ALGO, int STYLE, int U, bool COHERENT, bool NOQ = false, bool LOCAL = false>
__device__ __forceinline__ void relax_step(const Args &a, Xw &x, const Step<U> &s, RoundAcc &acc) {
    constexpr bool QUEUE = (STYLE == WORKLIST || STYLE == DELTA) && !NOQ;
    constexpr int WQ = QUEUE ? 256 : 1;
    const int lane = threadIdx.x & 31;
#ifdef FK_PROBE   // tools/expand_probe.cu: time the expansion without (0) / with (1) the gathers
    if (fk_probe_mode < 2) {
#pragma unroll
        for (int q = 0; q < U; q++) {
            if (!s.ok[q]) continue;
            const int32_t g = fk_probe_mode == 1 ? ld_value<COHERENT>(a.val + s.v[q], x.pl) : 0;
            if ((int32_t)(s.p[q] + (uint32_t)s.wt[q]) < g || s.v[q] == 0xfffffffeu) acc.nu++;
        }
        return;
    }
#endif
    if constexpr (STYLE == VFUSED) {
        // Fused partitioned round (SURVEY §8(e) "B200-native stretch"): the
        // relax kernel is the exchange.  Every target is filtered against
        // this part's OWN full-length value array (owned range: the values;
        // elsewhere: the smallest proposal this part has made -- a local
        // gather, never a remote one), lowered there, and a target owned by
        // another part also gets the proposal as a fire-and-forget RED.MIN
        // into the owner's value array and a RED.OR into the owner's round
        // bitmap -- over NVLink peer memory on real GPUs, device pointers when
        // simulated / loopback.  No exchange step or apply kernel follows.
        // A proposal the owner already beats only costs a redundant RED.
        static_assert(ALGO == SSSP, "fused rounds run SSSP (BFS as unit-weight SSSP)");
        int32_t cur[U];
#pragma unroll
        for (int q = 0; q < U; q++) cur[q] = s.ok[q] ? ld_value<COHERENT>(a.val + s.v[q], x.pl) : 0;
        const size_t boff = (size_t)(x.bm_now - a.bm0);   // this round's bitmap inside every part's bitmaps
#pragma unroll
        for (int q = 0; q < U; q++) {
            if (!s.ok[q]) continue;
            const uint32_t v = s.v[q];
            const uint32_t cand = s.p[q] + (uint32_t)s.wt[q];
            if (cand >= (uint32_t)INF) { acc.ovf = true; continue; }
            if ((int32_t)cand >= cur[q]) continue;
            atomicMin(a.val + v, (int32_t)cand);   // owned value or local shadow
            if (v >= a.lo && v < a.hi) {
                atomicOr(x.bm_now + (v >> 5), 1u << (v & 31));
            } else {
                int lo = 0, hi = (int)a.nparts;   // owner: largest o with bounds[o] <= v
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (a.bounds[mid] <= v) lo = mid; else hi = mid;
                }
                atomicMin(a.peer_val[lo] + v, (int32_t)cand);
                atomicOr(a.peer_bm[lo] + boff + (v >> 5), 1u << (v & 31));
                x.qn++;   // remote improvements of this lane (Ctrl::xremote)
            }
            acc.nu++; acc.chg = true;
        }
    } else {
    int32_t cur[U];
#pragma unroll
    for (int q = 0; q < U; q++) {
        cur[q] = 0;
        if (s.ok[q]) {
            if (ALGO == BFS) cur[q] = bit_test(a.vis, s.v[q]) ? 0 : INF;
            else cur[q] = ld_value<COHERENT>(a.val + s.v[q], x.pl);
        }
    }
    bool need[U];
    uint32_t citem[U];
#pragma unroll
    for (int q = 0; q < U; q++) {
        need[q] = false; citem[q] = 0;
        if (!s.ok[q]) continue;
        if (ALGO == SSSP) {
            const uint32_t cand = s.p[q] + (uint32_t)s.wt[q];
            if (cand >= (uint32_t)INF) {
                acc.ovf = true;
            } else if ((int32_t)cand < cur[q]) {
                atomicMin(a.val + s.v[q], (int32_t)cand);   // result unused: RED.MIN
                acc.nu++; acc.chg = true;
                if (STYLE == DELTA && cand >= x.thr) {   // beyond the bucket: park in the far set
                    atomicOr(a.vis + (s.v[q] >> 5), 1u << (s.v[q] & 31));
                    x.pend_min = cand < x.pend_min ? cand : x.pend_min;
                } else {
                    need[q] = true; citem[q] = s.v[q];
                }
            }
        } else if (ALGO == BFS) {
            // t.dist > lev+1 -> t.dist = lev+1 (plain store;
            // concurrent writers store the same value, R9)
            if (cur[q] == INF) {
                if (QUEUE) {   // the queue needs exactly-once: claim
                    need[q] = true; citem[q] = s.v[q];
                } else {   // VERTEX: the level is written when the vertex is expanded next round
                    if (!(is_vertex(STYLE) && x.lazy)) atomicOr(a.vis + (s.v[q] >> 5), 1u << (s.v[q] & 31));
                    atomicOr(x.bm_now + (s.v[q] >> 5), 1u << (s.v[q] & 31));
                    if (NOQ) put_level(a, s.v[q], x.lev + 1);
                    acc.nu++; acc.chg = true;
                }
            }
        }
    }
    if (!QUEUE) {
        if (ALGO == SSSP) {
#pragma unroll
            for (int q = 0; q < U; q++)
                if (need[q]) atomicOr(x.bm_now + (citem[q] >> 5), 1u << (citem[q] & 31));
            if (STYLE == DELTA) {   // no-queue DELTA round: count the near marks (bucket continues iff > 0)
#pragma unroll
                for (int q = 0; q < U; q++) x.qn += (uint32_t)__popc(__ballot_sync(FULL, need[q]));
            }
        }
    } else if (LOCAL) {
        static_assert(!LOCAL || ALGO == SSSP, "local continuation is min-relaxation (SSSP)");
#pragma unroll
        for (int q = 0; q < U; q++) {
            const unsigned mask = __ballot_sync(FULL, need[q]);
            if (need[q]) x.wq[x.qn + __popc(mask & ((1u << lane) - 1u))] = citem[q];
            x.qn += __popc(mask);
        }
        __syncwarp();
        if (x.qn > (uint32_t)(WQ - 32 * U)) {   // room for the next step: compact, else hand everything over
            const uint32_t cnt = x.qn - x.qh;
            if (x.qh >= 32 * U) {
                for (uint32_t i0 = 0; i0 < cnt; i0 += 32) {   // ascending chunks: writes stay below later reads
                    const uint32_t t = i0 + lane < cnt ? x.wq[x.qh + i0 + lane] : 0u;
                    __syncwarp();
                    if (i0 + lane < cnt) x.wq[i0 + lane] = t;
                    __syncwarp();
                }
                x.qh = 0; x.qn = cnt;
            } else {
                spill_local(a, x);
            }
        }
    } else {
        uint32_t got[U];
#pragma unroll
        for (int q = 0; q < U; q++) {
            got[q] = 0xffffffffu;
            if (!need[q]) continue;
            uint32_t *bmp = ALGO == BFS ? a.vis : x.bm_now;
            got[q] = atomicOr(bmp + (citem[q] >> 5), 1u << (citem[q] & 31));
        }
#pragma unroll
        for (int q = 0; q < U; q++) {
            const bool want = need[q] && !(got[q] & (1u << (citem[q] & 31)));
            if (ALGO == BFS && want) {
                put_level(a, citem[q], x.lev + 1);
                atomicOr(x.bm_now + (citem[q] >> 5), 1u << (citem[q] & 31));   // dense rounds read it
                acc.nu++; acc.chg = true;
            }
            const unsigned mask = __ballot_sync(FULL, want);
            if (want) x.wq[x.qn + __popc(mask & ((1u << lane) - 1u))] = citem[q];
            x.qn += __popc(mask);
        }
        __syncwarp();
        if (x.qn > (uint32_t)(WQ > 32 * U ? WQ - 32 * U : 0)) {   // flush the staged appends
            uint32_t b = 0;
            if (lane == 0) b = atomicAdd(&x.c->out_len, x.qn);
            b = __shfl_sync(FULL, b, 0);
            for (uint32_t i = lane; i < x.qn; i += 32) q_put(a, x.out, b + i, x.wq[i]);
            __syncwarp();
            x.qn = 0;
        }
    }
    }   // STYLE != VFUSED
}

// DELTA: an item at or beyond the (split) bucket threshold goes back to the far set.
__device__ __forceinline__ void park_far(const Args &a, Xw &x, uint32_t u, uint32_t d) {
    atomicOr(a.vis + (u >> 5), 1u << (u & 31));
    x.pend_min = d < x.pend_min ? d : x.pend_min;
}

// Relax the arcs of one 32-item tile (lane: value pay, arcs [beg, beg+deg)).
// Software pipeline ACROSS tiles: each step's (col, w) loads are issued, then
// the PREVIOUS step -- possibly of the previous tile -- gathers and relaxes.
// With average degree ~4 a tile is a single step, so a per-tile pipeline
// would expose two dependent latencies per tile (arcs, then gathered values;
// ncu: 43 % of the stall samples); here the arc loads of tile t are in flight
// while tile t-1's gathers are waited on.  The caller drains `pend` with
// relax_step at the end of the round.
template <int ALGO, int STYLE, int U, bool COHERENT, bool NOQ, bool LOCAL = false>
__device__ __forceinline__ void relax_tile(const Args &a, Xw &x, uint32_t beg, uint32_t deg, uint32_t pay,
                                           RoundAcc &acc, Step<U> &pend) {
    const int lane = threadIdx.x & 31;
    if (!COHERENT && x.hthr && deg > x.hthr) {   // a long row: expanded by the whole CTA (cta_heavy)
        const uint32_t slot = atomicAdd(x.hn, 1u);
        if (slot < HMAX) { x.hb[slot] = beg; x.hd[slot] = deg; x.hp[slot] = pay; deg = 0; }
    }
    uint32_t incl = deg;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
    }
    const uint32_t total = __shfl_sync(FULL, incl, 31);
    const uint32_t excl = incl - deg;
    if (lane == 0) acc.ne += total;
    for (uint32_t base = 0; base < total; base += 32 * U) {   // warp-uniform
        Step<U> nx;
        uint32_t e[U];
#pragma unroll
        for (int q = 0; q < U; q++) {
            const uint32_t k = base + q * 32 + lane;
            nx.ok[q] = k < total;
            int j = 0;
#pragma unroll
            for (int st = 16; st > 0; st >>= 1) {
                const uint32_t ex = __shfl_sync(FULL, excl, j + st);
                if (ex <= k) j += st;
            }
            const uint32_t bj = __shfl_sync(FULL, beg, j), xj = __shfl_sync(FULL, excl, j);
            nx.p[q] = __shfl_sync(FULL, pay, j);
            e[q] = bj + (k - xj);
        }
#pragma unroll
        for (int q = 0; q < U; q++) {
            nx.v[q] = 0; nx.wt[q] = 0;
            if (nx.ok[q]) {
                if (ALGO == SSSP) {   // one 8-byte (col, w) word
                    const uint2 w2 = ld_stream2(x.arcs + e[q], x.pf);
                    nx.v[q] = w2.x; nx.wt[q] = (int32_t)w2.y;
                } else {
                    nx.v[q] = ld_stream(a.col + e[q], x.pf);
                }
            }
        }
        if (pend.live) relax_step<ALGO, STYLE, U, COHERENT, NOQ, LOCAL>(a, x, pend, acc);
        pend = nx;
        pend.live = true;
    }
}

// CTA-level cooperative expansion (north_star item 3; the load imbalance of
// skewed degrees): the rows longer than x.hthr arcs that
// this CTA's warps met in the round were listed in shared memory
// (relax_tile); after every warp's own work all warps of the CTA walk them
// together, each row 32*U arcs per warp step, warps interleaved -- an RMAT
// hub or a star centre costs a CTA deg / (32 U W) steps instead of one warp
// deg / (32 U).  All arcs of a step belong to one row, so no search is
// needed.  Every thread of the CTA must call this (block barriers).
template <int ALGO, int STYLE, int U, bool NOQ, bool LOCAL>
__device__ __forceinline__ void cta_heavy(const Args &a, Xw &x, RoundAcc &acc) {
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint32_t nh = min(*x.hn, HMAX);
    Step<U> pend;
    pend.live = false;
    for (uint32_t h = 0; h < nh; h++) {
        const uint32_t beg = x.hb[h], deg = x.hd[h], pay = x.hp[h];
        if (threadIdx.x == 0) acc.ne += deg;
        for (uint32_t base = (uint32_t)wid * 32u * U; base < deg; base += (uint32_t)nw * 32u * U) {   // warp-uniform
            Step<U> nx;
#pragma unroll
            for (int q = 0; q < U; q++) {
                const uint32_t k = base + (uint32_t)q * 32u + lane;
                nx.ok[q] = k < deg;
                nx.p[q] = pay;
                nx.v[q] = 0; nx.wt[q] = 0;
                if (nx.ok[q]) {
                    if (ALGO == SSSP) {
                        const uint2 w2 = ld_stream2(x.arcs + beg + k, x.pf);
                        nx.v[q] = w2.x; nx.wt[q] = (int32_t)w2.y;
                    } else {
                        nx.v[q] = ld_stream(a.col + beg + k, x.pf);
                    }
                }
            }
            if (pend.live) relax_step<ALGO, STYLE, U, false, NOQ, LOCAL>(a, x, pend, acc);
            pend = nx;
            pend.live = true;
        }
    }
    if (pend.live) relax_step<ALGO, STYLE, U, false, NOQ, LOCAL>(a, x, pend, acc);
    __syncthreads();
    if (threadIdx.x == 0) *x.hn = 0;
}

// One round of expansion by this warp.  sit: the warp's 1024-entry shared
// item list (dense rounds).
template <int ALGO, int STYLE, int U, bool COHERENT, bool NOQ = false, bool LOCAL = false>
__device__ __forceinline__ void expand_round(const Args &a, Ctrl *c, uint32_t iter, uint32_t thr, const uint32_t *in,
                                             uint32_t *out, uint32_t nitems, bool dense, bool blocked, uint32_t *wq,
                                             uint32_t *sit, RoundAcc &acc, uint32_t ltiles = 0,
                                             uint32_t *heavy = nullptr) {
    constexpr bool QUEUE = STYLE == WORKLIST || STYLE == DELTA;
    const int lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t wstride = nwarps * 32;
    Xw x;
    x.bm_now = bm_of(a, iter); x.bm_prev = bm_of(a, iter - 1); x.out = out; x.wq = wq; x.c = c;
    x.lev = iter - 1; x.thr = thr; x.qh = 0; x.qn = 0; x.pend_min = 0xffffffffu;
    x.pf = pol_evict_first(); x.pl = pol_evict_last();
    x.lazy = ALGO == BFS && is_vertex(STYLE) && c->lazy;
    x.hthr = heavy && !COHERENT ? a.cta_thr : 0u;   // heavy: the CTA's shared long-row list
    if (x.hthr) { x.hn = heavy; x.hb = heavy + 1; x.hd = heavy + 1 + HMAX; x.hp = heavy + 1 + 2 * HMAX; }
    blocked = blocked && ALGO == SSSP && a.nblk > 1;
    const uint32_t K = blocked ? a.nblk : 1u;
    Step<U> pend;
    pend.live = false;

    for (uint32_t k = 0; k < K; k++) {
        const bool first = k == 0, last = k + 1 == K;
        x.rows = blocked ? a.rowb + (size_t)k * (a.n + 1) : a.row_off;
        x.arcs = blocked ? a.cwb : a.cw;
        if (dense) {
            auto word_at = [&](uint32_t wi) -> uint32_t {
                return wi < a.nwords ? (COHERENT ? __ldcg(x.bm_prev + wi) : x.bm_prev[wi]) : 0u;
            };
            // the bitmap words of the next DP groups are in flight (a light
            // round's groups are mostly empty: one load latency per DP groups)
            constexpr int DP = 4;
            uint32_t wq[DP];
#pragma unroll
            for (int k = 0; k < DP; k++) wq[k] = word_at(gw * 32 + k * wstride + lane);
            for (uint32_t g0 = gw * 32; g0 < a.nwords; g0 += wstride) {   // warp-uniform
                const uint32_t wi = g0 + lane;
                const uint32_t word0 = wq[0];
#pragma unroll
                for (int k = 0; k < DP - 1; k++) wq[k] = wq[k + 1];
                wq[DP - 1] = word_at(g0 + DP * wstride + lane);
                if (!__any_sync(FULL, word0 != 0u)) continue;
                if (QUEUE && last && word0) x.bm_prev[wi] = 0u;   // recycle the claim bitmap
                // skip_now: items already marked for the next round wait for it
                // (their expansion now would use a value the next one supersedes)
                uint32_t word = word0;
                if (ALGO == SSSP && a.skip_now && word) word &= ~(COHERENT ? __ldcg(x.bm_now + wi) : x.bm_now[wi]);
                const uint32_t cnt = __popc(word);
                uint32_t incl = cnt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(FULL, incl, o);
                    if (lane >= o) incl += y;
                }
                const uint32_t total = __shfl_sync(FULL, incl, 31);
                if (total == 0) continue;
                uint32_t pos = incl - cnt;
                for (uint32_t y = word; y; y &= y - 1) sit[pos++] = wi * 32u + (uint32_t)(__ffs(y) - 1);
                __syncwarp();
                uint32_t u1 = lane < total ? sit[lane] : NONE, pay1, beg1, end1;
                item_rows<ALGO, COHERENT>(a, x, u1, pay1, beg1, end1);
                for (uint32_t j0 = 0; j0 < total; j0 += 32) {   // warp-uniform
                    const uint32_t u = u1, pay = pay1, beg = beg1;
                    uint32_t deg = end1 - beg1;
                    u1 = j0 + 32 + lane < total ? sit[j0 + 32 + lane] : NONE;
                    item_rows<ALGO, COHERENT>(a, x, u1, pay1, beg1, end1);
                    if (u != NONE && first) {
                        acc.nv++;
                        if (ALGO == BFS && (is_vertex(STYLE) || (STYLE == WORKLIST && a.wl_pull)))
                            put_level(a, u, x.lev);   // discovered last round (WORKLIST: maybe by a pull round)
                    }
                    if (u == NONE || (ALGO == SSSP && pay == (uint32_t)INF)) deg = 0;
                    if (STYLE == DELTA && u != NONE && pay >= x.thr) {   // bucket was split: back to the far set
                        if (first) park_far(a, x, u, pay);
                        deg = 0;
                    }
                    relax_tile<ALGO, STYLE, U, COHERENT, NOQ>(a, x, beg, deg, pay, acc, pend);
                }
                __syncwarp();
            }
        } else {
            // software pipeline: u1 = item of the current tile, u2 = item of the next
            auto item_of = [&](uint32_t idx) -> uint32_t {
                return idx < nitems ? ld_item<COHERENT>(in + idx, x.pf) : NONE;
            };
            uint32_t wb = gw * 32;
            uint32_t u1 = item_of(wb + lane), u2 = item_of(wb + wstride + lane), pay1, beg1, end1;
            item_rows<ALGO, COHERENT>(a, x, u1, pay1, beg1, end1);
            for (; wb < nitems; wb += wstride) {   // warp-uniform
                const uint32_t u = u1, pay = pay1, beg = beg1;
                uint32_t deg = end1 - beg1;
                u1 = u2;
                u2 = item_of(wb + 2 * wstride + lane);
                item_rows<ALGO, COHERENT>(a, x, u1, pay1, beg1, end1);
                if (QUEUE && last && u != NONE) x.bm_prev[u >> 5] = 0u;   // recycle the claim bitmap
                if (u != NONE && first) acc.nv++;
                if (u == NONE || (ALGO == SSSP && pay == (uint32_t)INF)) deg = 0;
                if (ALGO == SSSP && a.skip_now && deg &&
                    (((COHERENT ? __ldcg(x.bm_now + (u >> 5)) : x.bm_now[u >> 5]) >> (u & 31)) & 1u))
                    deg = 0;   // queued again already: expanded next round with its newer value
                if (STYLE == DELTA && u != NONE && pay >= x.thr) {   // bucket was split: back to the far set
                    if (first) park_far(a, x, u, pay);
                    deg = 0;
                }
                relax_tile<ALGO, STYLE, U, COHERENT, NOQ, LOCAL>(a, x, beg, deg, pay, acc, pend);
            }
        }
    }
    if (pend.live) relax_step<ALGO, STYLE, U, COHERENT, NOQ, LOCAL>(a, x, pend, acc);   // drain the pipeline
    if constexpr (!COHERENT) {
        if (x.hthr) cta_heavy<ALGO, STYLE, U, NOQ, LOCAL>(a, x, acc);   // before the local continuation: its stacks
    }
    if constexpr (LOCAL) {
        // Local continuation: the warp expands the targets it improved itself,
        // 32 at a time, up to ltiles tiles, instead of leaving each hop to
        // a round of its own (road graphs: thousands of rounds of a few
        // thousand items, each round bound by launch and dependent-access
        // latency).  Any relaxation order reaches the same least fixpoint
        // (R8); values written in this kernel are read L1-bypassing
        // (COHERENT), so every expansion sees the value that pushed it or a
        // lower one.
        pend.live = false;
        for (uint32_t t = 0; t < ltiles && x.qn > x.qh; t++) {   // warp-uniform
            const uint32_t take = min(x.qn - x.qh, 32u);
            const uint32_t u = lane < take ? x.wq[x.qh + lane] : NONE;
            __syncwarp();
            x.qh += take;
            uint32_t pay, beg, end;
            item_rows<ALGO, true>(a, x, u, pay, beg, end);
            uint32_t deg = end - beg;
            if (u != NONE) acc.nv++;
            if (u == NONE || pay == (uint32_t)INF) deg = 0;
            relax_tile<ALGO, STYLE, U, true, NOQ, LOCAL>(a, x, beg, deg, pay, acc, pend);
            if (pend.live) relax_step<ALGO, STYLE, U, true, NOQ, LOCAL>(a, x, pend, acc);
            pend.live = false;
        }
        spill_local(a, x);
    }
    if (QUEUE && !NOQ && !LOCAL) {
        __syncwarp();
        if (x.qn) {
            uint32_t b = 0;
            if (lane == 0) b = atomicAdd(&c->out_len, x.qn);
            b = __shfl_sync(FULL, b, 0);
            for (uint32_t i = lane; i < x.qn; i += 32) q_put(a, out, b + i, wq[i]);
            __syncwarp();
        }
    }
    if (STYLE == VFUSED) {   // remote improvements sent this round, one atomic per warp
        unsigned long long r = x.qn;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(FULL, r, o);
        if (lane == 0 && r) atomicAdd(&c->xremote, r);
    }
    if (STYLE == DELTA && NOQ) {   // near marks of a no-queue round: the next round's frontier size (upper bound)
        if (lane == 0 && x.qn) atomicAdd(&c->out_len, x.qn);
    }
    if (STYLE == DELTA) {   // warp-min, one atomicMin per warp
        uint32_t pm = x.pend_min;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint32_t y = __shfl_xor_sync(FULL, pm, o);
            pm = y < pm ? y : pm;
        }
        if (lane == 0 && pm != 0xffffffffu) atomicMin(&c->minpend, pm);
    }
    if (acc.ovf) c->cand_ovf = 1;
}

// One round per launch (VERTEX, and the queue styles when not persistent).
template <int ALGO, int STYLE, int B, int U, int MINB>
__global__ void __launch_bounds__(B, MINB) k_expand_warp(Args a) {
    static_assert(is_vertex(STYLE) || STYLE == WORKLIST || STYLE == DELTA, "expand is for VERTEX/WORKLIST/DELTA");
    constexpr int WQ = (STYLE == WORKLIST || STYLE == DELTA) ? 256 : 1;
    Ctrl *c = a.ctrl;
    if (c->done || (ALGO == BFS && (is_vertex(STYLE) || STYLE == WORKLIST) && c->pull)) return;
    if (STYLE == DELTA && c->mode != MODE_NEAR) {   // this round refills the near queue from the far set
        unsigned long long nv = 0;
        scan_far_round<false>(a, c, c->iter, c->thr, c->sel ? a.fr0 : a.fr1, nv);
        flush_counters<B>(a, nv, 0ull, 0ull, false, false);
        return;
    }
    const uint32_t iter = c->iter;
    // (BFS WORKLIST with pull rounds: a pull round leaves its input bitmap
    // unrecycled, so every round clears the one after next like VERTEX)
    if (is_vertex(STYLE) || (ALGO == BFS && STYLE == WORKLIST && a.wl_pull)) clear_next_bitmap(a, iter);
    const uint32_t thr = STYLE == DELTA ? c->thr : 0xffffffffu;
    const uint32_t *in = c->sel ? a.fr1 : a.fr0;
    uint32_t *out = c->sel ? a.fr0 : a.fr1;
    const uint32_t nitems = c->in_len;
    const bool dense = is_vertex(STYLE) || (a.dense_div && nitems > a.n / a.dense_div);
    const bool blocked = is_vertex(STYLE) ? c->blk != 0 : (a.blk_div && nitems > a.n / a.blk_div);
    __shared__ uint32_t s_q[B / 32][WQ];
    __shared__ uint32_t s_it[B / 32][1024];
    __shared__ uint32_t s_heavy[1 + 3 * HMAX];   // count, then beg / deg / pay of the CTA's long rows
    if (threadIdx.x == 0) s_heavy[0] = 0u;
    __syncthreads();
    RoundAcc acc;
    if ((STYLE == WORKLIST && dense && a.wl_noq) || (STYLE == DELTA && dense && a.dl_noq)) {
        // dense WORKLIST / DELTA round: items from the bitmap, improved vertices
        // marked in the next bitmap with reductions -- no claim atomics, no
        // queue (DELTA: near targets only; far ones are parked as usual).  The
        // next round reads its items from that bitmap (Ctrl::prevnoq); if it is
        // sparse, it builds the queue again with claims.
        if (blockIdx.x == 0 && threadIdx.x == 0) c->noq = 1;
        expand_round<ALGO, STYLE, U, false, true>(a, c, iter, thr, in, out, nitems, true, blocked,
                                                  s_q[threadIdx.x >> 5], s_it[threadIdx.x >> 5], acc, 0, s_heavy);
    } else if (ALGO == SSSP && (STYLE == DELTA ? a.local_tiles && nitems <= a.local_max && !c->prevnoq
                                               : a.wl_local_tiles && nitems <= a.wl_local_max && !c->prevnoq) &&
               !dense && !blocked) {
        // sparse SSSP rounds with local continuation (expand_round)
        expand_round<ALGO, STYLE, U, false, false, ALGO == SSSP>(
            a, c, iter, thr, in, out, nitems, false, false, s_q[threadIdx.x >> 5], s_it[threadIdx.x >> 5], acc,
            STYLE == DELTA ? a.local_tiles : a.wl_local_tiles, s_heavy);
    } else {
        expand_round<ALGO, STYLE, U, false>(a, c, iter, thr, in, out, nitems,
                                            dense || ((STYLE == WORKLIST || STYLE == DELTA) && c->prevnoq), blocked,
                                            s_q[threadIdx.x >> 5], s_it[threadIdx.x >> 5], acc, 0, s_heavy);
    }
    if (STYLE == VFUSED) __threadfence_system();   // remote REDs performed before the termination collective
    flush_counters<B>(a, acc.nv, acc.ne, acc.nu, acc.chg, acc.ovf);
}

// ------------------------------------------------------------------ EDGE style (COO)
// Per quad of four consecutive arcs whose sources' activity bits
// (bm[(r-1)%3], L1/L2-resident) are in actmask: col/w are fetched only for
// quads with an active source.
template <int ALGO>
__device__ __forceinline__ void edge_quad(const Args &a, uint32_t q, const uint32_t (&s)[4], uint32_t actmask,
                                          uint32_t m4, uint32_t tail, uint32_t lev, uint32_t *bm_now, uint64_t pf,
                                          uint64_t pl, unsigned long long &ne, unsigned long long &nu, bool &chg,
                                          bool &ovf) {
    uint32_t d[4] = {0, 0, 0, 0}, pay[4] = {0, 0, 0, 0};
    int32_t ww[4] = {0, 0, 0, 0};
    if (q < m4) {
        if (ALGO == SSSP) {
            const uint4 x0 = ld_stream4(a.cwb + 4ull * q, pf), x1 = ld_stream4(a.cwb + 4ull * q + 2, pf);
            d[0] = x0.x; ww[0] = (int32_t)x0.y; d[1] = x0.z; ww[1] = (int32_t)x0.w;
            d[2] = x1.x; ww[2] = (int32_t)x1.y; d[3] = x1.z; ww[3] = (int32_t)x1.w;
        } else {
            const uint4 d4 = ld_stream4(a.col + 4ull * q, pf);
            d[0] = d4.x; d[1] = d4.y; d[2] = d4.z; d[3] = d4.w;
        }
    } else {
        for (uint32_t j = 0; j < tail; j++) {
            if (ALGO == SSSP) {
                const uint2 x = ld_stream2(a.cwb + 4ull * q + j, pf);
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
                put_level(a, d[j], lev + 1);
                atomicOr(bm_now + (d[j] >> 5), 1u << (d[j] & 31));
                nu++; chg = true;
            }
        }
    }
}

// EDGE style (COO).  A warp owns chunks of ECH = 128*QP
// consecutive arcs (lane: QP quads, 16-byte loads, consecutive lanes on
// consecutive quads).  Each chunk's source range [lo, hi] is precomputed at
// load time (k_chunk_range), so liveness needs no src[] read: the warp checks
// 32 chunks at once, one per lane (range -> the range's activity-bitmap words
// -> ballot), and expands only the live ones -- a sparse round streams a few
// bitmap words per 128 sources instead of 4 bytes of src[] per arc.  In a live
// chunk every arc's source bit is tested and (col, w) fetched only for quads
// with an active source.
template <int ALGO, int QP>
__device__ __forceinline__ void edge_load_src(const uint32_t *srcp, uint32_t ch, uint32_t m4, uint32_t nq,
                                              uint32_t tail, uint64_t pf, uint32_t (&sq)[QP][4]) {
    constexpr uint32_t ECH = 128u * QP;
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int p = 0; p < QP; p++) {
        const uint32_t q = ch * (ECH / 4) + p * 32 + lane;
        sq[p][0] = sq[p][1] = sq[p][2] = sq[p][3] = 0;
        if (q < m4) {
            const uint4 s4 = ld_stream4(srcp + 4ull * q, pf);
            sq[p][0] = s4.x; sq[p][1] = s4.y; sq[p][2] = s4.z; sq[p][3] = s4.w;
        } else if (q < nq) {
            for (uint32_t j = 0; j < tail; j++) sq[p][j] = ld_stream(srcp + 4ull * q + j, pf);
        }
    }
}

#ifndef EDGE_PREFETCH
#define EDGE_PREFETCH 1
#endif
template <int ALGO, int B, int QP>
__global__ void __launch_bounds__(B) k_edge(Args a) {
    static_assert(ALGO != CC, "CC has its own EDGE kernel (cc.cuh)");
    constexpr uint32_t ECH = 128u * QP;
    Ctrl *c = a.ctrl;
    if (c->done) return;
    const uint32_t iter = c->iter, lev = iter - 1;
    clear_next_bitmap(a, iter);
    const uint32_t *bm_prev = bm_of(a, iter - 1);
    uint32_t *bm_now = bm_of(a, iter);
    const uint64_t pf = pol_evict_first(), pl = pol_evict_last();
    const uint32_t m4 = a.m >> 2, tail = a.m & 3u;
    const uint32_t nq = m4 + (tail ? 1u : 0u);
    const uint32_t *srcp = ALGO == SSSP ? a.srcb : a.src;   // SSSP: destination-blocked arc order
    const uint2 *rng = ALGO == SSSP ? a.chunkb : a.chunk;
    const int lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * B + threadIdx.x) >> 5, nwarps = (gridDim.x * B) >> 5;
    const uint32_t nch = (a.m + ECH - 1) / ECH;
    unsigned long long ne = 0, nu = 0;
    bool chg = false, ovf = false;
    for (uint32_t cb = gw; cb < nch; cb += 32 * nwarps) {   // warp-uniform: 32 chunks, one per lane
        const uint32_t myc = cb + lane * nwarps;
        bool live = false;
        if (myc < nch) {
            const uint2 r = rng[myc];
            const uint32_t w0 = r.x >> 5, nw = (r.y >> 5) - w0 + 1;
            if (nw > 32) {
                live = true;
            } else {   // a 512-arc chunk spans ~9 words on rand-25M's blocked order, up to 32 checked
                uint32_t any = 0;
#pragma unroll 8
                for (uint32_t k = 0; k < nw; k++) any |= bm_prev[w0 + k];
                live = any != 0;
            }
        }
        unsigned mask = __ballot_sync(FULL, live);
        if (!mask) continue;
        uint32_t sq[QP][4];
        uint32_t ch = cb + (__ffs(mask) - 1) * nwarps;
        mask &= mask - 1;
        edge_load_src<ALGO, QP>(srcp, ch, m4, nq, tail, pf, sq);
        for (;;) {   // warp-uniform over the live chunks of the batch
            // the next live chunk's sources are loaded while this one is relaxed
            const uint32_t chn = mask ? cb + (__ffs(mask) - 1) * nwarps : NONE;
            mask &= mask - 1;
            uint32_t sqn[QP][4];
            if (EDGE_PREFETCH && chn != NONE) edge_load_src<ALGO, QP>(srcp, chn, m4, nq, tail, pf, sqn);
            uint32_t act[QP];
#pragma unroll
            for (int p = 0; p < QP; p++) {
                const uint32_t q = ch * (ECH / 4) + p * 32 + lane;
                const uint32_t cntq = q < m4 ? 4u : (q < nq ? tail : 0u);
                act[p] = 0;
#pragma unroll
                for (int j = 0; j < 4; j++)   // the source must be active (improved / discovered last round)
                    if ((uint32_t)j < cntq && bit_test(bm_prev, sq[p][j])) act[p] |= 1u << j;
            }
#pragma unroll
            for (int p = 0; p < QP; p++)
                if (act[p])
                    edge_quad<ALGO>(a, ch * (ECH / 4) + p * 32 + lane, sq[p], act[p], m4, tail, lev, bm_now, pf, pl,
                                    ne, nu, chg, ovf);
            if (chn == NONE) break;
            ch = chn;
            if (EDGE_PREFETCH) {
#pragma unroll
                for (int p = 0; p < QP; p++)
#pragma unroll
                    for (int j = 0; j < 4; j++) sq[p][j] = sqn[p][j];
            } else {
                edge_load_src<ALGO, QP>(srcp, ch, m4, nq, tail, pf, sq);
            }
        }
    }
    flush_counters<B>(a, 0ull, ne, nu, chg, ovf);
}

// Source range [min, max] of every ECH-arc chunk of a COO source array (one
// warp per chunk; load time).
__global__ void k_chunk_range(uint32_t m, uint32_t ech, const uint32_t *src, uint2 *rng) {
    const int lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t nch = (m + ech - 1) / ech;
    for (uint32_t ch = gw; ch < nch; ch += nwarps) {
        uint32_t lo = 0xffffffffu, hi = 0;
        const uint32_t e1 = (ch + 1) * ech < m ? (ch + 1) * ech : m;
        for (uint32_t e = ch * ech + lane; e < e1; e += 32) {
            const uint32_t u = src[e];
            lo = u < lo ? u : lo;
            hi = u > hi ? u : hi;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = min(lo, __shfl_xor_sync(FULL, lo, o));
            hi = max(hi, __shfl_xor_sync(FULL, hi, o));
        }
        if (lane == 0) rng[ch] = make_uint2(lo, hi);
    }
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
// Direction of the next BFS VERTEX round (direction-optimising BFS): 0 push
// (top-down over the frontier's out-arcs), 1 / 2 pull (bottom-up over the
// unvisited vertices' in-arcs; 2 = the compacted form for a sparse unvisited
// set).  Estimated L2 requests of each (random 32-byte sectors; the measured
// cost unit of every relax kernel here), from F = the new
// frontier, U = unvisited vertices, d = arcs per item of this push round (or
// m/n after a pull round) and m_f = F d:
//   push ~ m_f (a visited-bit gather per arc) + 2F (row offsets and arcs of
//          each frontier vertex) + 2.5 x expected discoveries
//          U (1 - exp(-m_f / n)) (visited and frontier REDs, level store),
//   pull ~ 2U (in-arc offsets and first in-arcs of each unvisited vertex)
//          + U min(m/n, m/m_f) (in-arcs scanned until a parent: 1/p with
//          p = m_f/m the frontier's share of the in-arcs).
// rule 1 / 2 (option pull_rule) keeps the round-1 rule instead -- pull iff
// F > n / pull_div -- with the word / compacted form.  Only the schedule
// changes, never the levels.
__device__ __forceinline__ uint32_t bfs_direction(const Ctrl *c, uint32_t n, uint64_t m, uint32_t pull_div,
                                                  uint32_t rule) {
    if (!pull_div || c->found == 0) return 0;
    if (rule == 1 || rule == 2) return c->found > n / pull_div ? rule : 0u;
    const float F = (float)c->found, U = c->visited >= n ? 0.f : (float)(n - c->visited), N = (float)n, M = (float)m;
    if (c->found <= n / 1024u) return 0;   // small frontier: push
    const float d = !c->pull && c->rnd_items ? (float)c->rnd_edges / (float)c->rnd_items : M / N;
    const float mf = F * d;
    const float push = mf + 2.f * F + 2.5f * U * (1.f - __expf(-mf / N));
    const float pull = 2.f * U + U * fminf(M / N, mf > 0.f ? M / mf : M / N);
    if (pull >= push) return 0;
    return U * 2.f < N ? 2u : 1u;
}

// Decides on the device whether another round runs ("if
// (changed == 0) break" / SPEC.md:221 "worklist non-empty"), and drives the
// CUDA-graph WHILE node through cudaGraphSetConditional.
// aux_div: BFS VERTEX: pull_div (bottom-up threshold); DELTA: split_div (bucket split)
template <int ALGO, int STYLE>
__device__ __forceinline__ bool advance_step(Ctrl *c, uint32_t launches_per_round, uint32_t n, uint32_t aux_div,
                                             uint32_t blk_div, uint32_t rule = 0, uint64_t m = 0,
                                             uint32_t lazy_div = 0) {
    const uint32_t pull_div = aux_div;
    if (c->done) return false;
    if (c->status == ST_QUEUE) { c->done = 1; return false; }
    c->launches += launches_per_round;
    bool more = STYLE == WORKLIST ? (c->noq ? c->changed != 0 : c->out_len > 0) : c->changed != 0;
    if (STYLE == DELTA) {
        if (c->mode == MODE_SCAN) {
            more = true;                 // the refilled near queue (possibly empty) comes next
            c->mode = MODE_NEAR;
        } else if (c->out_len == 0) {    // bucket exhausted: move T to the next non-empty bucket
            more = c->minpend != 0xffffffffu;
            c->bk_items += c->in_len;
            c->bk_rounds++;
            if (c->delta_adapt) {
                // Adaptive Δ (auto mode): a round costs a fixed ~10 µs of launch
                // and dependent-latency time, worth ~10^5 relaxed items.  A
                // bucket whose rounds averaged fewer items was latency-bound:
                // double Δ (fewer, fuller rounds; road grids).  One whose
                // rounds averaged millions relaxed many vertices more than
                // once: halve Δ, not below the initial width.  Any sequence
                // of thresholds reaches the same fixpoint (T always moves past
                // the smallest parked distance).
                const unsigned long long avg = c->bk_items / (c->bk_rounds ? c->bk_rounds : 1u);
                // (growth capped at delta_cap x the initial width: on a road grid
                // the rounds stay small whatever Δ, and a larger Δ only adds work)
                if (avg < (128ull << 10) && (uint64_t)c->delta < (uint64_t)c->delta_cap * c->delta0 &&
                    c->delta < (1u << 26))
                    c->delta *= 2u;
                else if (avg > (2ull << 20) && c->delta / 2u >= c->delta0) c->delta /= 2u;
            }
            c->bk_items = 0;
            c->bk_rounds = 0;
            if (more) {
                const uint64_t t = ((uint64_t)c->minpend / c->delta + 1) * c->delta;
                c->thr = t > 0x7fffffffull ? 0x7fffffffu : (uint32_t)t;
                c->minpend = 0xffffffffu;   // recomputed by the far scan and later parkings
                c->mode = MODE_SCAN;
                c->noq = 0;                 // the refill round builds a queue
            }
        } else {
            more = true;
            c->bk_items += c->in_len;   // a near round of the current bucket
            c->bk_rounds++;
            // bucket split (aux_div = DELTA's split_div): a near round that
            // hands on more than n / split_div items relaxes many vertices
            // before their final value is known -- halve the bucket (not below
            // the initial width); items of the next round at or above the new
            // threshold are parked in the far set when loaded (expand_round)
            if (c->delta_adapt && aux_div && c->out_len > n / aux_div && c->delta / 2u >= c->delta0) {
                c->delta /= 2u;
                c->thr -= c->delta;
            }
        }
    }
    if (c->status != ST_OK) more = false;
    if (more && c->iter >= c->cap) { c->status = ST_NOT_CONVERGED; more = false; }
    if (more) {
        c->iter++;
        c->changed = 0;
        if (STYLE == WORKLIST || (STYLE == DELTA && c->mode == MODE_NEAR)) {
            // after a no-queue round the frontier size is estimated by the
            // filter passes (>= the improved vertices): it only decides dense
            c->in_len = STYLE == WORKLIST && c->noq ? c->found : c->out_len;
            if (ALGO == BFS && STYLE == WORKLIST && pull_div) {   // bottom-up rounds (option wl_pull)
                c->visited += c->noq ? c->found : c->out_len;   // (no-queue rounds: marks, an over-count)
                c->found = c->noq ? c->found : c->out_len;
                c->pull = bfs_direction(c, n, m, pull_div, rule);
                c->rnd_items = 0;
                c->rnd_edges = 0;
            }
            c->prevnoq = c->noq;
            c->noq = 0;
            c->out_len = 0;
            c->sel ^= 1u;
            c->all_active = 0;
        } else if (STYLE == VERTEX) {
            c->in_len = 0;   // VERTEX rounds read the activity bitmap
            // direction-optimising BFS: bottom-up while the next frontier is large
            if (ALGO == BFS) {
                // a lazy round counted a vertex once per marking arc; the round
                // after it counted them exactly while merging them into vis
                if (c->merge) c->visited = c->visited - c->lazy_found + c->exact;
                c->visited += c->found;
                c->merge = c->lazy;   // a lazy round's discoveries join vis in the next round's k_pull
                c->lazy_found = c->found;
                c->exact = 0;
                c->pull = bfs_direction(c, n, m, pull_div, rule);
                c->lazy = !c->pull && lazy_div && c->found > n / lazy_div;
                c->rnd_items = 0;
                c->rnd_edges = 0;
            }
            // SSSP: the next round walks the destination-blocked layout when this
            // round improved many vertices (its frontier is large)
            c->blk = blk_div && c->found > n / blk_div;
        }
        c->found = 0;
    } else {
        c->done = 1;
    }
    return more;
}

// Decides on the device whether another round runs ("if
// (changed == 0) break" / SPEC.md:221 "worklist non-empty"), and drives the
// CUDA-graph WHILE node through cudaGraphSetConditional.
template <int ALGO, int STYLE>
__global__ void k_advance(Ctrl *c, cudaGraphConditionalHandle h, int in_graph, uint32_t launches_per_round,
                          uint32_t n, uint32_t pull_div, uint32_t blk_div, uint32_t rule, uint32_t m,
                          uint32_t lazy_div) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const bool more = advance_step<ALGO, STYLE>(c, launches_per_round, n, pull_div, blk_div, rule, m, lazy_div);
    if (in_graph) cudaGraphSetConditional(h, more ? 1u : 0u);
}

// ------------------------------------------------------------------ persistent rounds
// Optional (FALCON_PERSIST=1): queue styles (WORKLIST, DELTA) run their SMALL
// rounds (frontier <= max_items) inside one cooperative kernel: a round's
// expansion, then a grid barrier whose last arriving CTA performs the advance
// (the same advance_step as k_advance) and releases the others.  Large rounds
// leave the kernel and run as one launch per round; the CUDA-graph round body
// is [k_persist, round kernels, k_advance].  Data written earlier in the
// kernel is read with L1-bypassing loads.  Measured on B200 a persistent
// round costs about as much as a graph-launched one (~11-13 µs on the road
// grid: the round is bound by its chain of dependent memory accesses, the
// barrier is ~2.7 µs, tools/barrier_probe.cu), so it is off by default.
__device__ __forceinline__ uint32_t ldv(const uint32_t *p) { return *reinterpret_cast<const volatile uint32_t *>(p); }

template <int ALGO, int STYLE>
__device__ __forceinline__ void grid_barrier_advance(Ctrl *c, uint32_t n, uint32_t pull_div, uint32_t blk_div) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t gen = ldv(&c->bar_gen);
        __threadfence();
        const uint32_t arrived = atomicAdd(&c->bar_arrive, 1u);
        if (arrived == gridDim.x - 1) {
            c->bar_arrive = 0;
            advance_step<ALGO, STYLE>(c, 0u, n, STYLE == WORKLIST && ALGO == BFS ? 0u : pull_div, blk_div);   // (no bottom-up rounds here)
            __threadfence();
            atomicExch(&c->bar_gen, gen + 1u);
        } else {
            while (ldv(&c->bar_gen) == gen) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

template <int ALGO, int STYLE, int B, int U>
__global__ void __launch_bounds__(B, 2) k_persist(Args a, uint32_t pull_div, uint32_t max_items) {
    static_assert(STYLE == WORKLIST || STYLE == DELTA, "persistent rounds are for the queue styles");
    __shared__ uint32_t s_q[B / 32][256];
    Ctrl *c = a.ctrl;
    RoundAcc acc;
    for (;;) {
        // uniform exits (every CTA reads the same state after the same barrier):
        // done, or a frontier large enough for the one-launch-per-round kernels
        if (ldv(&c->done)) break;
        const bool scan = STYLE == DELTA && ldv(&c->mode) == MODE_SCAN;
        if (!scan && ldv(&c->in_len) > max_items) break;
        if ((STYLE == WORKLIST || STYLE == DELTA) && ldv(&c->prevnoq)) break;   // frontier only in the bitmap
        const uint32_t iter = ldv(&c->iter), sel = ldv(&c->sel);
        const uint32_t thr = STYLE == DELTA ? ldv(&c->thr) : 0xffffffffu;
        const uint32_t *in = sel ? a.fr1 : a.fr0;
        uint32_t *out = sel ? a.fr0 : a.fr1;
        if (scan)
            scan_far_round<true>(a, c, iter, thr, out, acc.nv);
        else
            expand_round<ALGO, STYLE, U, true>(a, c, iter, thr, in, out, ldv(&c->in_len), false, false,
                                               s_q[threadIdx.x >> 5], nullptr, acc);
        grid_barrier_advance<ALGO, STYLE>(c, a.n, pull_div, a.blk_div);
    }
    flush_counters<B>(a, acc.nv, acc.ne, acc.nu, acc.chg, acc.ovf);
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

// Overflow certificate (reading R3, run only when some candidate d[u]+w
// reached INF during the fixpoint).  A candidate >= INF is never applied, so
// every vertex whose least fixpoint distance is < INF still gets it exactly
// (all prefixes of its shortest path stay below INF); a vertex reachable only
// by paths of length >= INF stays at INF.  The oracle's overflow condition
// (a finite shortest distance >= INF) is therefore equivalent to: some arc
// u -> v has final val[u] < INF and final val[v] == INF -- schedule-free.
// Rows may be a part's (empty outside its owned range); val is the full array.
__global__ void k_overflow_check(uint32_t n, const uint32_t *row_off, const uint32_t *col, const int32_t *val,
                                 int *flag) {
    const uint32_t stride = gridDim.x * blockDim.x;
    bool bad = false;
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < n && !bad; u += stride) {
        if (val[u] == INF) continue;
        const uint32_t e1 = row_off[u + 1];
        for (uint32_t e = row_off[u]; e < e1; e++)
            if (val[col[e]] == INF) { bad = true; break; }
    }
    if (bad) atomicOr(flag, 1);
}

__global__ void k_interleave(uint64_t m, const uint32_t *col, const int32_t *w, uint2 *cw) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride)
        cw[e] = make_uint2(col[e], (uint32_t)w[e]);
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
__global__ void k_fill_i32(int32_t *p, uint64_t len, int32_t x) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += stride) p[i] = x;
}

// Destination-blocked layout, built once per graph: block k
// holds the arcs whose target lies in [k*bsz, (k+1)*bsz), as its own CSR over
// all sources, rows in source order and arcs in their original order.  One
// row per thread (rows are short; an RMAT hub row takes one thread µs).
constexpr uint32_t MAX_BLK = 16;
__global__ void k_blk_count(uint32_t n, const uint32_t *row_off, const uint32_t *col, uint32_t bsz, uint32_t nblk,
                            uint32_t *cnt) {
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint64_t ld = (uint64_t)n + 1;
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += stride) {
        uint32_t c[MAX_BLK];
        for (uint32_t k = 0; k < nblk; k++) c[k] = 0;
        const uint32_t e1 = row_off[u + 1];
        for (uint32_t e = row_off[u]; e < e1; e++) c[col[e] / bsz]++;
        for (uint32_t k = 0; k < nblk; k++) cnt[k * ld + u] = c[k];
    }
    if (blockIdx.x == 0 && threadIdx.x < nblk) cnt[threadIdx.x * ld + n] = 0;
}
// Blocked layout by sorting (ensure_blocked): block id of every arc's target
// and the identity permutation, then the gather of the sorted order.
__global__ void k_blk_keys(uint64_t m, const uint32_t *col, uint32_t bsz, uint8_t *keys, uint32_t *perm) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
        keys[e] = (uint8_t)(col[e] / bsz);
        perm[e] = (uint32_t)e;
    }
}
__global__ void k_blk_gather(uint64_t m, const uint32_t *perm, const uint2 *cw, const uint32_t *src, uint2 *cwb,
                             uint32_t *srcb) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
        const uint32_t e = perm[i];
        cwb[i] = cw[e];
        srcb[i] = src[e];
    }
}

// Offsets of a CSR whose m arcs have the sorted targets key[]: off[v] = first
// position with key >= v, off[n] = m.  Thread i fills the offsets of the
// targets in (key[i-1], key[i]].
__global__ void k_rin_off(uint64_t m, uint32_t n, const uint32_t *key, uint32_t *off) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= m; i += stride) {
        const uint32_t lo = i == 0 ? 0u : key[i - 1] + 1u;
        const uint32_t hi = i == m ? n : key[i];
        for (uint32_t v = lo; v <= hi; v++) off[v] = (uint32_t)i;
    }
}

// COO sources in CSR order: src[e] = u for every arc of row u (row-parallel
// fill; rows are short except RMAT hubs, which one thread writes in µs).
__global__ void k_build_src(uint32_t n, uint32_t m, const uint32_t *row_off, uint32_t *src) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += stride) {
        const uint32_t e1 = row_off[u + 1];
        for (uint32_t e = row_off[u]; e < e1; e++) src[e] = u;
    }
}

}  // namespace fk
