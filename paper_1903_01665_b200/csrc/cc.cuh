// cc.cuh -- connected components (weak) by min-label hooking with pointer
// jumping, as a lock-free union-find (readings R6 / R15).
//
// label[] starts as the identity (CC is "propagation based";
// SPEC.md:452 min-label convention).  For an arc (u, v) the two roots are
// found by pointer jumping (path splitting on the way), and the LARGER root
// is hooked under the smaller one with a compare-and-swap that only succeeds
// on a root.  Every non-root therefore points to a smaller id, every root is
// the minimum of its tree, and after all arcs are processed and every label
// compressed to its root, label[v] = min vertex id of v's weak component --
// the unique result the oracle computes.  One pass over the arcs suffices
// (the hook phase never has to be repeated), unlike label propagation whose
// rounds grow with the diameter ("Falcon does not perform well
// on road inputs" for CC).
//
// Styles: VERTEX walks each vertex's CSR row (warp-cooperative), EDGE walks
// the COO arcs, WORKLIST is sampling-then-worklist (two rounds hooking each
// vertex to its first two out-neighbours, then only the vertices outside
// the largest component process all their in- and out-arcs).
#pragma once
#include "kernels.cuh"

namespace fk {

// root of x; path splitting: every visited node is pointed at its
// grandparent (benign races: any written value is an ancestor)
__device__ __forceinline__ uint32_t uf_find(int32_t *L, uint32_t x) {
    uint32_t cur = (uint32_t)L[x];
    if (cur == x) return x;
    uint32_t prev = x;
    for (;;) {
        const uint32_t nxt = (uint32_t)L[cur];
        if (nxt == cur) return cur;
        L[prev] = (int32_t)nxt;
        prev = cur;
        cur = nxt;
    }
}

// hook the larger root under the smaller; retry while the CAS loses a race
__device__ __forceinline__ bool uf_unite(int32_t *L, uint32_t a, uint32_t b) {
    a = uf_find(L, a);
    b = uf_find(L, b);
    bool hooked = false;
    while (a != b) {
        if (a > b) { const uint32_t t = a; a = b; b = t; }
        const uint32_t old = atomicCAS(reinterpret_cast<unsigned *>(L + b), b, a);
        if (old == b) { hooked = true; break; }
        b = uf_find(L, old);   // b was hooked meanwhile: continue from its new root
    }
    return hooked;
}

// VERTEX: warp-cooperative walk over all vertices' out-arcs (same shuffle
// scan / binary search as k_expand_warp), unite(u, v) per arc.
// MAXD > 0: only the first MAXD arcs of every row (WORKLIST sampling, R15).
template <int B, int MAXD = 0>
__global__ void __launch_bounds__(B) k_cc_vertex(Args a) {
    if (a.ctrl->done) return;
    const int lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * B + threadIdx.x) >> 5, nwarps = (gridDim.x * B) >> 5;
    const uint64_t pf = pol_evict_first();
    unsigned long long nv = 0, ne = 0, nu = 0;
    for (uint32_t wb = gw * 32; wb < a.n; wb += nwarps * 32) {
        const uint32_t u = wb + lane;
        uint32_t beg = 0, deg = 0;
        if (u < a.n) {
            beg = ld_ro(a.row_off + u);
            deg = ld_ro(a.row_off + u + 1) - beg;
            if (MAXD > 0 && deg > (uint32_t)MAXD) deg = MAXD;
            nv++;
        }
        uint32_t incl = deg;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t total = __shfl_sync(FULL, incl, 31), excl = incl - deg;
        if (lane == 0) ne += total;
        for (uint32_t base = 0; base < total; base += 32) {
            const uint32_t k = base + lane;
            int j = 0;
#pragma unroll
            for (int st = 16; st > 0; st >>= 1) {
                const uint32_t ex = __shfl_sync(FULL, excl, j + st);
                if (ex <= k) j += st;
            }
            const uint32_t bj = __shfl_sync(FULL, beg, j), xj = __shfl_sync(FULL, excl, j);
            const uint32_t uj = wb + (uint32_t)j;
            if (k < total) {
                const uint32_t v = ld_stream(a.col + bj + (k - xj), pf);
                if (uf_unite(a.val, uj, v)) nu++;
            }
        }
    }
    flush_counters<B>(a, nv, ne, nu, nu != 0, false);   // `changed` = some hook (partitioned rounds)
}

// EDGE: one arc per thread per step over the COO arrays (coalesced src/col
// loads; a full-occupancy grid keeps ~2K independent find chains per SM)
template <int B>
__global__ void __launch_bounds__(B) k_cc_edge(Args a) {
    const uint64_t pf = pol_evict_first();
    unsigned long long ne = 0, nu = 0;
    const uint32_t stride = gridDim.x * B;
    uint32_t e = blockIdx.x * B + threadIdx.x;
    // the next arc's endpoints are loaded while this arc's find chains run
    uint32_t u = e < a.m ? ld_stream(a.src + e, pf) : 0u, v = e < a.m ? ld_stream(a.col + e, pf) : 0u;
    for (; e < a.m; e += stride) {
        const uint32_t en = e + stride;
        const uint32_t un = en < a.m ? ld_stream(a.src + en, pf) : 0u, vn = en < a.m ? ld_stream(a.col + en, pf) : 0u;
        ne++;
        if (uf_unite(a.val, u, v)) nu++;
        u = un;
        v = vn;
    }
    flush_counters<B>(a, 0ull, ne, nu, false, false);
}

// The label of the largest component, estimated from 1024 hashed samples
// (mode of their roots).  One CTA of 1024 threads.  Correctness does not
// depend on the estimate: it only decides which vertices may skip.
__global__ void k_cc_giant(Args a) {
    constexpr int S = 1024;   // Afforest samples 1024: the mode is the giant whenever one exists
    __shared__ uint32_t s_lab[S];
    __shared__ unsigned long long s_best;
    if (threadIdx.x == 0) s_best = 0;
    for (int i = threadIdx.x; i < S; i += blockDim.x) {
        uint32_t h = (uint32_t)i * 0x9E3779B9u + 0x7F4A7C15u;
        h ^= h >> 16; h *= 0x85EBCA6Bu; h ^= h >> 13;
        s_lab[i] = uf_find(a.val, h % a.n);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < S; i += blockDim.x) {
        uint32_t cnt = 0;
        const uint32_t x = s_lab[i];
        for (int j = 0; j < S; j++) cnt += s_lab[j] == x;
        atomicMax(&s_best, ((unsigned long long)cnt << 32) | (0xffffffffu - x));
    }
    __syncthreads();
    if (threadIdx.x == 0) a.ctrl->source = 0xffffffffu - (uint32_t)(s_best & 0xffffffffu);   // giant label
}

// WORKLIST, final round: the vertices whose root is not the giant label
// (compacted on the fly, warp-cooperatively) unite with ALL their out- and
// in-neighbours; arcs between two giant vertices need no work.
template <int B>
__global__ void __launch_bounds__(B) k_cc_rest(Args a) {
    const int lane = threadIdx.x & 31;
    const uint32_t giant = a.ctrl->source;
    const uint32_t gw = (blockIdx.x * B + threadIdx.x) >> 5, nwarps = (gridDim.x * B) >> 5;
    const uint64_t pf = pol_evict_first();
    unsigned long long nv = 0, ne = 0, nu = 0;
    for (uint32_t wb = gw * 32; wb < a.n; wb += nwarps * 32) {
        const uint32_t u = wb + lane;
        uint32_t ob = 0, od = 0, ib = 0, id = 0;
        if (u < a.n && uf_find(a.val, u) != giant) {
            ob = ld_ro(a.row_off + u); od = ld_ro(a.row_off + u + 1) - ob;
            ib = ld_ro(a.rin_off + u); id = ld_ro(a.rin_off + u + 1) - ib;
            nv++;
        }
        const uint32_t deg = od + id;
        uint32_t incl = deg;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t total = __shfl_sync(FULL, incl, 31), excl = incl - deg;
        if (total == 0) continue;
        if (lane == 0) ne += total;
        for (uint32_t base = 0; base < total; base += 32) {
            const uint32_t k = base + lane;
            int j = 0;
#pragma unroll
            for (int st = 16; st > 0; st >>= 1) {
                const uint32_t ex = __shfl_sync(FULL, excl, j + st);
                if (ex <= k) j += st;
            }
            const uint32_t xj = __shfl_sync(FULL, excl, j), obj = __shfl_sync(FULL, ob, j),
                           odj = __shfl_sync(FULL, od, j), ibj = __shfl_sync(FULL, ib, j);
            if (k < total) {
                const uint32_t r = k - xj;
                const uint32_t v = r < odj ? ld_stream(a.col + obj + r, pf) : ld_stream(a.rin_col + ibj + (r - odj), pf);
                if (uf_unite(a.val, wb + (uint32_t)j, v)) nu++;
            }
        }
    }
    flush_counters<B>(a, nv, ne, nu, false, false);
}

}  // namespace fk
