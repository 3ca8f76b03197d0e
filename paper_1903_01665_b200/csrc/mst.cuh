// mst.cuh -- minimum spanning forest by Borůvka rounds (SURVEY.md §8(f)
// row 4; the paper's MST, Table 2
// "Boruvka with single-guarded component merging").
//
// Every arc u->v is the undirected edge {u, v}.  comp[] (the graph's value
// array) holds, at the start of a round, each vertex's component root.  A
// round:
//   1. min:   every arc whose endpoints lie in different components proposes
//             key = (w << 32) | arc index to BOTH components with a 64-bit
//             atomicMin (VERTEX: CSR rows, warp-cooperative; EDGE: COO arcs).
//             The key is a strict total order, so each component's choice is
//             unique and the chosen edges form a forest plus mutual pairs.
//   2. hook:  every root c with a choice e points at the component across e;
//             of a mutual pair (both chose e) the smaller id stays a root.
//             Each hooking root adds w(e) once to the forest weight -- the
//             paper's `single`-guarded merge, here a choice
//             that only one side of an edge can make.
//   3. apply the new parents, then pointer-jump (k_compress) every vertex to
//             its root.
// Rounds repeat until no root hooks (at most log2(n) rounds: every component
// merges with at least one other each round).  Labels are finally mapped to
// the minimum vertex id of each tree (= the CC label).
#pragma once
#include "kernels.cuh"

namespace fk {

constexpr unsigned long long MST_NONE = ~0ull;

__device__ __forceinline__ void mst_propose(unsigned long long *best, uint32_t cu, uint32_t cv, unsigned long long key) {
    if (cu == cv) return;   // inside one tree: never again useful
    if (key < __ldcg(best + cu)) atomicMin(best + cu, key);
    if (key < __ldcg(best + cv)) atomicMin(best + cv, key);
}

// reset the choices; thread 0 also clears the round's hook count
__global__ void k_mst_reset(Args a, unsigned long long *best) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < a.n; v += stride) best[v] = MST_NONE;
    if (blockIdx.x == 0 && threadIdx.x == 0) { a.ctrl->hooks = 0; a.ctrl->out_len = 0; a.ctrl->found = 0; }
}

// Live items: counted per thread (folded into Ctrl::found by the CTA's
// counter flush) and, when out != NULL, appended warp-aggregated to out.
__device__ __forceinline__ void mst_append(const Args &a, uint32_t *out, bool keep, uint32_t item,
                                           unsigned long long &nlive) {
    nlive += keep ? 1u : 0u;
    if (!out) return;
    const int lane = threadIdx.x & 31;
    const unsigned mask = __ballot_sync(FULL, keep);
    if (!mask) return;
    uint32_t b = 0;
    if (lane == 0) b = atomicAdd(&a.ctrl->out_len, (uint32_t)__popc(mask));
    b = __shfl_sync(FULL, b, 0);
    if (keep) out[b + __popc(mask & ((1u << lane) - 1u))] = item;
}

// VERTEX: warp-cooperative walk over every vertex's CSR row (the shuffle
// scan / binary search of k_expand_warp); one component lookup per vertex.
// Items: the vertices of `in` (nin of them), or every vertex when in == NULL
// (first round).  A vertex with at least one arc leaving its component is
// kept for the next round (`out`): a row whose arcs all lie inside one tree
// never proposes again (trees only merge).
template <int B>
__global__ void __launch_bounds__(B) k_mst_min_vertex(Args a, unsigned long long *best, const uint32_t *in,
                                                      uint32_t nin, uint32_t *out) {
    __shared__ uint32_t s_live[B / 32][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t gw = (blockIdx.x * B + threadIdx.x) >> 5, nwarps = (gridDim.x * B) >> 5;
    const uint64_t pf = pol_evict_first();
    unsigned long long ne = 0, nlive = 0;
    const uint32_t nitems = in ? nin : a.n;
    for (uint32_t wb = gw * 32; wb < nitems; wb += nwarps * 32) {
        const uint32_t u = wb + lane < nitems ? (in ? in[wb + lane] : wb + lane) : NONE;
        s_live[wid][lane] = 0;
        uint32_t beg = 0, deg = 0, cu = 0;
        if (u != NONE) {
            beg = ld_ro(a.row_off + u);
            deg = ld_ro(a.row_off + u + 1) - beg;
            cu = (uint32_t)__ldcg(a.val + u);
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
            const uint32_t cj = __shfl_sync(FULL, cu, j);
            if (k < total) {
                const uint32_t e = bj + (k - xj);
                const uint2 x = ld_stream2(a.cw + e, pf);
                const uint32_t cv = (uint32_t)__ldcg(a.val + x.x);
                if (cv != cj) s_live[wid][j] = 1u;   // benign race: every writer stores 1
                mst_propose(best, cj, cv, ((unsigned long long)x.y << 32) | e);
            }
        }
        __syncwarp();
        mst_append(a, out, u != NONE && s_live[wid][lane], u, nlive);
        __syncwarp();
    }
    flush_counters<B>(a, 0ull, ne, nlive, false, false);   // nlive -> Ctrl::found
}

// EDGE: the arcs of `in` (nin arc indices), or all arcs (four per thread,
// 16-byte loads) when in == NULL (first round).  Arcs still leaving their
// component are kept for the next round (`out`).
template <int B>
__global__ void __launch_bounds__(B) k_mst_min_edge(Args a, unsigned long long *best, const uint32_t *in,
                                                    uint32_t nin, uint32_t *out) {
    const uint64_t pf = pol_evict_first();
    unsigned long long ne = 0, nlive = 0;
    const uint32_t stride = gridDim.x * B;
    const uint32_t nitems = in ? nin : a.m;
    const uint32_t n4 = (nitems + 3) >> 2;
    for (uint32_t q = blockIdx.x * B + threadIdx.x; q - threadIdx.x % 32 < n4; q += stride) {   // warp-uniform
        uint32_t e[4], s[4], d[4], w[4];
        bool ok[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const uint32_t i = 4 * q + j;
            ok[j] = q < n4 && i < nitems;
            e[j] = ok[j] ? (in ? ld_stream(in + i, pf) : i) : 0u;
        }
        if (!in && 4 * q + 3 < nitems) {   // full scan: 16-byte loads of four consecutive arcs
            const uint4 s4 = ld_stream4(a.src + 4ull * q, pf);
            const uint4 x0 = ld_stream4(a.cw + 4ull * q, pf), x1 = ld_stream4(a.cw + 4ull * q + 2, pf);
            s[0] = s4.x; s[1] = s4.y; s[2] = s4.z; s[3] = s4.w;
            d[0] = x0.x; w[0] = x0.y; d[1] = x0.z; w[1] = x0.w; d[2] = x1.x; w[2] = x1.y; d[3] = x1.z; w[3] = x1.w;
        } else {
#pragma unroll
            for (int j = 0; j < 4; j++) {
                s[j] = d[j] = w[j] = 0;
                if (!ok[j]) continue;
                s[j] = ld_ro(a.src + e[j]);
                const uint2 x = ld_stream2(a.cw + e[j], pf);
                d[j] = x.x; w[j] = x.y;
            }
        }
        uint32_t cs[4], cd[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
            cs[j] = ok[j] ? (uint32_t)__ldcg(a.val + s[j]) : 0u;
            cd[j] = ok[j] ? (uint32_t)__ldcg(a.val + d[j]) : 0u;
        }
#pragma unroll
        for (int j = 0; j < 4; j++) {
            if (ok[j]) {
                ne++;
                mst_propose(best, cs[j], cd[j], ((unsigned long long)w[j] << 32) | e[j]);
            }
            mst_append(a, out, ok[j] && cs[j] != cd[j], e[j], nlive);
        }
    }
    flush_counters<B>(a, 0ull, ne, nlive, false, false);   // nlive -> Ctrl::found
}

// Every root with a choice points at the component across it (nxt); the
// smaller root of a mutual pair stays.  Hooking roots add the edge weight.
template <int B>
__global__ void __launch_bounds__(B) k_mst_hook(Args a, const unsigned long long *best, uint32_t *nxt) {
    unsigned long long wsum = 0;
    uint32_t hooks = 0;
    const uint32_t stride = gridDim.x * B;
    for (uint32_t v = blockIdx.x * B + threadIdx.x; v < a.n; v += stride) {
        if ((uint32_t)a.val[v] != v) continue;   // not a root
        const unsigned long long k = best[v];
        uint32_t to = v;
        if (k != MST_NONE) {
            const uint32_t e = (uint32_t)k;
            const uint32_t cs = (uint32_t)a.val[a.src[e]], cd = (uint32_t)a.val[a.cw[e].x];
            const uint32_t other = cs == v ? cd : cs;
            const bool mutual = best[other] == k;
            if (!(mutual && v < other)) {
                to = other;
                wsum += k >> 32;
                hooks++;
            }
        }
        nxt[v] = to;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        wsum += __shfl_xor_sync(FULL, wsum, o);
        hooks += __shfl_xor_sync(FULL, hooks, o);
    }
    if ((threadIdx.x & 31) == 0 && hooks) {
        atomicAdd(&a.ctrl->wsum, wsum);
        atomicAdd(&a.ctrl->hooks, hooks);
        atomicAdd(&a.ctrl->updates, (unsigned long long)hooks);
    }
}

__global__ void k_mst_apply(Args a, const uint32_t *nxt) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < a.n; v += stride)
        if ((uint32_t)a.val[v] == v) a.val[v] = (int32_t)nxt[v];
}

// Final labels: the minimum vertex id of each tree (minid reuses best[] as u32).
__global__ void k_mst_minid(Args a, uint32_t *minid) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < a.n; v += stride) atomicMin(minid + a.val[v], v);
}
__global__ void k_mst_label(Args a, const uint32_t *minid) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < a.n; v += stride) a.val[v] = (int32_t)minid[a.val[v]];
}

}  // namespace fk
