// partition.cuh -- 1-D vertex-partitioned multi-GPU path (DESIGN.md §7,
// SURVEY.md §8(e)).  Included by falcon.cu (needs falcon_graph, load, run).
//
// Part q owns vertices [bounds[q], bounds[q+1]) -- contiguous ranges chosen
// by EDGE count (binary search on the row_off prefix), or the slices the
// ranks pass (FALCON_LOAD_SLICE) -- and stores the CSR rows of its owned
// vertices only (global column ids), plus a full-length value array: the
// owned range is authoritative, the rest holds this part's proposals for
// remote vertices (the "shadow").  A superstep:
//   1. relax: the single-GPU VERTEX round (k_expand_warp) over the
//      part's rows; MIN lands in the local full-length array;
//   2. exchange, one of
//      - fused (the default between ranks): the relax kernel itself sends
//        every remote improvement as a RED.MIN + bitmap RED.OR into the
//        owner's arrays over peer memory (NVLink; CUDA IPC mappings), so no
//        exchange step follows;
//      - dense: every owner receives the MIN over all parts of its range
//        (grouped ncclReduce(ncclMin), one per owner -- volume 4n(P-1)/P per
//        rank, the reduce-scatter of SURVEY §8(e)), then applies it;
//      - sparse: (vertex, value) pairs of the remote improvements, grouped
//        ncclSend / ncclRecv after a count exchange (host-synchronised per
//        superstep: the payload sizes are host arguments);
//   3. termination: ncclAllReduce(SUM) of the per-part `changed` flag, then
//      the usual device-side advance -- every part takes the same decision.
//      The host looks at the control block once every HOST_CHECK_EVERY
//      supersteps (fused and dense rounds have no per-superstep host sync).
// MIN is associative, commutative and idempotent, so any partition and any
// exchange schedule reach the same unique fixpoint: results are bit-identical
// to one GPU.  BFS runs as unit-weight SSSP (hop distance = level).  CC hooks
// on a replicated label array: local union-find pass, ncclAllReduce(MIN) of
// the parent array, pointer jumping, until no part hooks.
//
// Communicators: NCCL ranks (one process per GPU; libnccl bound at run time
// with dlopen, so single-GPU users never need it); LOOPBACK ranks (host
// threads of one process sharing a device, loopback.cuh: the same per-rank
// code with the NCCL calls served in-process -- how the rank path is tested
// on a one-GPU box); SIMULATED communicators (one handle runs all P parts on
// one device with device-kernel exchanges).
#pragma once
#include <dlfcn.h>
#include <nccl.h>

namespace {

// ------------------------------------------------------------------ NCCL binding
struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                           cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi *nccl_api() {
    static NcclApi api;
    static bool tried = false;
    if (tried) return api.h ? &api : nullptr;
    tried = true;
    const char *names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char *nm : names)
        if ((api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!api.h) return nullptr;
#define SYM(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(api.h, "nccl" #f))
    SYM(GetUniqueId); SYM(CommInitRank); SYM(CommDestroy); SYM(Reduce); SYM(AllReduce);
    SYM(Broadcast); SYM(GroupStart); SYM(GroupEnd); SYM(GetErrorString); SYM(Send); SYM(Recv); SYM(AllGather);
#undef SYM
    if (!api.GetUniqueId || !api.CommInitRank || !api.Reduce || !api.AllReduce || !api.Broadcast ||
        !api.GroupStart || !api.GroupEnd) {
        api.h = nullptr;
        return nullptr;
    }
    return &api;
}

}  // namespace

#include "loopback.cuh"

struct falcon_comm {
    int nranks = 1, rank = 0, device = 0;
    int simulated = 0;            // > 0: number of parts simulated on one device
    ncclComm_t nccl = nullptr;
    NcclApi *api = nullptr;       // libnccl, or the in-process loopback transport
    bool loopback = false;        // ranks are threads of this process on one device
};

namespace {

// The loopback transport behind the NCCL function table (loopback.cuh).
NcclApi *loopback_api() {
    static NcclApi api = [] {
        NcclApi a;
        a.h = reinterpret_cast<void *>(1);
        a.GetUniqueId = lb_GetUniqueId; a.CommInitRank = lb_CommInitRank; a.CommDestroy = lb_CommDestroy;
        a.Reduce = lb_Reduce; a.AllReduce = lb_AllReduce; a.Broadcast = lb_Broadcast; a.Send = lb_Send;
        a.Recv = lb_Recv; a.AllGather = lb_AllGather; a.GroupStart = lb_GroupStart; a.GroupEnd = lb_GroupEnd;
        a.GetErrorString = lb_GetErrorString;
        return a;
    }();
    return &api;
}

const char *nc_errstr(ncclResult_t r) {
    NcclApi *a = nccl_api();
    return a && a->GetErrorString ? a->GetErrorString(r) : lb_GetErrorString(r);
}

#define NC(call)                                                                                    \
    do {                                                                                            \
        ncclResult_t _r = (call);                                                                   \
        if (_r != ncclSuccess) return fail(FALCON_ERR_COMM, "%s: %s", #call, nc_errstr(_r));        \
    } while (0)

// ------------------------------------------------------------------ kernels
// apply: owned values lowered by a remote proposal become active
__global__ void k_apply_owned(Args a, const int32_t *recv, uint32_t lo, uint32_t cnt) {
    Ctrl *c = a.ctrl;
    if (c->done) return;
    uint32_t *bm_now = bm_of(a, c->iter);
    bool chg = false;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += stride) {
        const int32_t r = recv[i];
        const uint32_t v = lo + i;
        if (r < a.val[v]) {
            a.val[v] = r;
            atomicOr(bm_now + (v >> 5), 1u << (v & 31));
            chg = true;
        }
    }
    if (__syncthreads_or(chg) && threadIdx.x == 0) c->changed = 1;
}

// simulated exchange: recv of owner q = MIN over parts of vals[p][lo..hi)
__global__ void k_sim_reduce_min(const int32_t *const *vals, int nparts, uint32_t lo, uint32_t cnt, int32_t *recv) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += stride) {
        int32_t m = vals[0][lo + i];
        for (int p = 1; p < nparts; p++) m = min(m, vals[p][lo + i]);
        recv[i] = m;
    }
}

// simulated all-reduce(MIN) of the full arrays, written back to every part
__global__ void k_sim_allreduce_min(int32_t *const *vals, int nparts, uint32_t n) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        int32_t m = vals[0][i];
        for (int p = 1; p < nparts; p++) m = min(m, vals[p][i]);
        for (int p = 0; p < nparts; p++) vals[p][i] = m;
    }
}

// simulated all-reduce(SUM) of the parts' `changed` flags
__global__ void k_sim_sum_changed(Ctrl *const *ctrls, int nparts) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    uint32_t s = 0;
    for (int p = 0; p < nparts; p++) s += ctrls[p]->changed;
    for (int p = 0; p < nparts; p++) ctrls[p]->changed = s;
}

// ------------------------------------------------------------------ sparse exchange
// The remote vertices a part improved in this round are exactly the bits of
// bm[iter % 3] outside its owned range [lo, hi).  When their (vertex, value)
// pairs -- 8 bytes each -- are fewer bytes than the dense reduce-scatter
// (4 n (P-1) / P per rank), only they travel; MIN is idempotent, so a round
// may use either exchange.

__device__ __forceinline__ int owner_of(const uint32_t *bounds, int P, uint32_t v) {
    int lo = 0, hi = P;   // largest q with bounds[q] <= v
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (bounds[mid] <= v) lo = mid; else hi = mid;
    }
    return lo;
}

// counts[q] = remote improved vertices owned by q (PACK: also write the pairs
// into outbox[bounds[q] + slot]); one word per thread, aggregated per word
template <bool PACK>
__global__ void k_remote_pairs(Args a, uint32_t lo, uint32_t hi, const uint32_t *bounds, int P, uint32_t *counts,
                               uint2 *outbox) {
    Ctrl *c = a.ctrl;
    if (c->done) return;
    const uint32_t *bm_now = bm_of(a, c->iter);
    const uint32_t nw = (a.n + 31) / 32, stride = gridDim.x * blockDim.x;
    for (uint32_t wi = blockIdx.x * blockDim.x + threadIdx.x; wi < nw; wi += stride) {
        uint32_t word = bm_now[wi];
        if (!word) continue;
        const uint32_t vb = wi * 32;
        // drop the owned bits and the bits past n
        for (uint32_t b = 0; b < 32; b++) {
            const uint32_t v = vb + b;
            if (v >= a.n || (v >= lo && v < hi)) word &= ~(1u << b);
        }
        while (word) {   // runs of bits with one owner
            const uint32_t v0 = vb + (uint32_t)(__ffs(word) - 1);
            const int q = owner_of(bounds, P, v0);
            const uint32_t qend = bounds[q + 1];
            uint32_t sub = word;
            if (qend < vb + 32) sub &= (qend > vb ? ((1u << (qend - vb)) - 1u) : 0u);
            word &= ~sub;
            const uint32_t k = (uint32_t)__popc(sub);
            const uint32_t slot = atomicAdd(counts + q, k);
            if (PACK) {
                uint32_t i = 0;
                for (uint32_t y = sub; y; y &= y - 1, i++) {
                    const uint32_t v = vb + (uint32_t)(__ffs(y) - 1);
                    outbox[bounds[q] + slot + i] = make_uint2(v, (uint32_t)a.val[v]);
                }
            }
        }
    }
}

// statistics (simulated): pairs packed this round, summed over every part
__global__ void k_sum_counts(const uint32_t *const *counts, int P, unsigned long long *total) {
    unsigned long long t = 0;
    for (int i = threadIdx.x; i < P * P; i += blockDim.x) t += counts[i / P][i % P];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(FULL, t, o);
    if ((threadIdx.x & 31) == 0 && t) atomicAdd(total, t);
}

// owner side: apply received pairs (atomicMin, mark improved)
__global__ void k_apply_pairs(Args a, const uint2 *pairs, uint32_t cnt) {
    Ctrl *c = a.ctrl;
    if (c->done) return;
    uint32_t *bm_now = bm_of(a, c->iter);
    bool chg = false;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += stride) {
        const uint2 p = pairs[i];
        if ((int32_t)p.y < a.val[p.x] && (int32_t)p.y < atomicMin(a.val + p.x, (int32_t)p.y)) {
            atomicOr(bm_now + (p.x >> 5), 1u << (p.x & 31));
            chg = true;
        }
    }
    if (__syncthreads_or(chg) && threadIdx.x == 0) c->changed = 1;
}

// simulated: owner q applies every part's pairs for q straight from their outboxes
__global__ void k_sim_apply_pairs(Args a, const uint2 *const *outboxes, const uint32_t *const *counts, int P, int q,
                                  uint32_t qlo) {
    Ctrl *c = a.ctrl;
    if (c->done) return;
    uint32_t *bm_now = bm_of(a, c->iter);
    bool chg = false;
    for (int p = 0; p < P; p++) {
        if (p == q) continue;
        const uint32_t cnt = counts[p][q];
        const uint2 *pairs = outboxes[p] + qlo;
        const uint32_t stride = gridDim.x * blockDim.x;
        for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += stride) {
            const uint2 x = pairs[i];
            if ((int32_t)x.y < a.val[x.x] && (int32_t)x.y < atomicMin(a.val + x.x, (int32_t)x.y)) {
                atomicOr(bm_now + (x.x >> 5), 1u << (x.x & 31));
                chg = true;
            }
        }
    }
    if (__syncthreads_or(chg) && threadIdx.x == 0) c->changed = 1;
}

// ------------------------------------------------------------------ host side
// Boundaries of nparts contiguous vertex ranges with ~m/nparts arcs each:
// boundary q is the vertex v >= bounds[q-1] whose prefix row_off[v] is
// nearest to q*m/nparts (so part sizes deviate by at most one row's degree).
void partition_bounds(int64_t n, const uint32_t *row_off, int nparts, int64_t *bounds) {
    const uint64_t m = row_off[n];
    bounds[0] = 0;
    for (int q = 1; q < nparts; q++) {
        const uint64_t target = (m * (uint64_t)q) / (uint64_t)nparts;
        int64_t lo = bounds[q - 1], hi = n;   // smallest v >= bounds[q-1] with row_off[v] >= target
        while (lo < hi) {
            const int64_t mid = lo + (hi - lo) / 2;
            if (row_off[mid] < target) lo = mid + 1; else hi = mid;
        }
        if (lo > bounds[q - 1] && target - row_off[lo - 1] < (uint64_t)row_off[lo] - target) lo--;
        bounds[q] = lo;
    }
    bounds[nparts] = n;
}

void destroy(falcon_graph *g);

void destroy_partitioned(falcon_graph *g) {
    for (auto *p : g->parts) {
        cudaSetDevice(p->device);
        if (p->stream) cudaStreamSynchronize(p->stream);
        dfree(p->recv);
        dfree(p->cw_unit);
        p->recv = nullptr;
        p->cw_unit = nullptr;
        destroy(p);
    }
    g->parts.clear();
    dfree(g->bounds_d); dfree(g->d_outboxes); dfree(g->d_counts); dfree(g->xpairs_d);
    g->bounds_d = nullptr; g->d_outboxes = nullptr; g->d_counts = nullptr; g->xpairs_d = nullptr;
    for (void *q : g->ipc_opened) cudaIpcCloseMemHandle(q);
    g->ipc_opened.clear();
    dfree(g->d_peer_val); dfree(g->d_peer_bm);
    g->d_peer_val = nullptr; g->d_peer_bm = nullptr;
}

// The part bounds on the device (sparse and fused exchanges).
falcon_status_t ensure_bounds(falcon_graph *g) {
    if (g->bounds_d) return FALCON_OK;
    falcon_comm *cm = g->comm;
    const int P = cm->simulated ? cm->simulated : cm->nranks;
    cudaStream_t s = g->parts[0]->stream;
    std::vector<uint32_t> hb((size_t)P + 1);
    for (int q = 0; q <= P; q++) hb[(size_t)q] = (uint32_t)g->bounds[(size_t)q];
    CU(dmalloc(&g->bounds_d, (size_t)P + 1));
    CU(dmalloc(&g->xpairs_d, 1));
    CU(cudaMemsetAsync(g->xpairs_d, 0, 8, s));   // cached blocks are not zeroed
    CU(cudaMemcpyAsync(g->bounds_d, hb.data(), (size_t)(P + 1) * 4, cudaMemcpyHostToDevice, s));
    CU(cudaStreamSynchronize(s));
    return FALCON_OK;
}

// Peer tables of the fused exchange: every part's value array and round
// bitmaps.  Simulated parts and loopback ranks (one process, one device):
// plain device pointers (all-gathered between loopback ranks).  NCCL ranks:
// CUDA IPC handles of each rank's arrays, all-gathered over NCCL and opened
// with peer access, so a relax kernel's RED.MIN / RED.OR land directly in the
// owner's memory over NVLink.  A rank that cannot map a peer fails with COMM
// (auto mode then falls back to the dense exchange).
falcon_status_t ensure_fused(falcon_graph *g) {
    if (g->d_peer_val) return FALCON_OK;
    falcon_status_t st = ensure_bounds(g);
    if (st != FALCON_OK) return st;
    falcon_comm *cm = g->comm;
    const int P = cm->simulated ? cm->simulated : cm->nranks;
    cudaStream_t s = g->parts[0]->stream;
    std::vector<int32_t *> hv((size_t)P);
    std::vector<uint32_t *> hb((size_t)P);
    if (cm->simulated) {
        for (int q = 0; q < P; q++) { hv[(size_t)q] = g->parts[(size_t)q]->val; hb[(size_t)q] = g->parts[(size_t)q]->bm; }
    } else if (cm->loopback) {
        falcon_graph *me = g->parts[0];
        uint64_t mine[2] = {(uint64_t)(uintptr_t)me->val, (uint64_t)(uintptr_t)me->bm};
        uint64_t *d_send = nullptr, *d_all = nullptr;
        CU(dmalloc(&d_send, 2));
        CU(dmalloc(&d_all, 2 * (size_t)P));
        CU(cudaMemcpyAsync(d_send, mine, sizeof mine, cudaMemcpyHostToDevice, s));
        NC(cm->api->AllGather(d_send, d_all, 2, ncclUint64, cm->nccl, s));
        std::vector<uint64_t> all(2 * (size_t)P);
        CU(cudaMemcpyAsync(all.data(), d_all, sizeof(uint64_t) * 2 * P, cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        dfree(d_send); dfree(d_all);
        for (int q = 0; q < P; q++) {
            hv[(size_t)q] = reinterpret_cast<int32_t *>((uintptr_t)all[2 * (size_t)q]);
            hb[(size_t)q] = reinterpret_cast<uint32_t *>((uintptr_t)all[2 * (size_t)q + 1]);
        }
    } else {
        NcclApi *nc = cm->api;
        if (!nc->AllGather) return fail(FALCON_ERR_COMM, "ncclAllGather unavailable");
        falcon_graph *me = g->parts[0];
        cudaIpcMemHandle_t mine[2];
        CU(cudaIpcGetMemHandle(&mine[0], me->val));
        CU(cudaIpcGetMemHandle(&mine[1], me->bm));
        uint8_t *d_send = nullptr, *d_all = nullptr;
        CU(dmalloc(&d_send, sizeof mine));
        CU(dmalloc(&d_all, sizeof mine * (size_t)P));
        CU(cudaMemcpyAsync(d_send, mine, sizeof mine, cudaMemcpyHostToDevice, s));
        NC(nc->AllGather(d_send, d_all, sizeof mine, ncclUint8, cm->nccl, s));
        std::vector<cudaIpcMemHandle_t> all((size_t)P * 2);
        CU(cudaMemcpyAsync(all.data(), d_all, sizeof mine * (size_t)P, cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        dfree(d_send); dfree(d_all);
        for (int q = 0; q < P; q++) {
            if (q == cm->rank) { hv[(size_t)q] = me->val; hb[(size_t)q] = me->bm; continue; }
            void *pv = nullptr, *pb = nullptr;
            if (cudaIpcOpenMemHandle(&pv, all[(size_t)q * 2], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
                cudaIpcOpenMemHandle(&pb, all[(size_t)q * 2 + 1], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                cudaGetLastError();
                if (pv) cudaIpcCloseMemHandle(pv);
                return fail(FALCON_ERR_COMM, "rank %d cannot map rank %d's memory (no peer access)", cm->rank, q);
            }
            g->ipc_opened.push_back(pv);
            g->ipc_opened.push_back(pb);
            hv[(size_t)q] = static_cast<int32_t *>(pv);
            hb[(size_t)q] = static_cast<uint32_t *>(pb);
        }
    }
    CU(dmalloc(&g->d_peer_val, (size_t)P));
    CU(dmalloc(&g->d_peer_bm, (size_t)P));
    CU(cudaMemcpyAsync(g->d_peer_val, hv.data(), sizeof(int32_t *) * P, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(g->d_peer_bm, hb.data(), sizeof(uint32_t *) * P, cudaMemcpyHostToDevice, s));
    CU(cudaStreamSynchronize(s));
    return FALCON_OK;
}

// Buffers of the sparse exchange, allocated on first use.
falcon_status_t ensure_sparse(falcon_graph *g) {
    if (g->parts[0]->xcounts) return FALCON_OK;
    falcon_status_t st0 = ensure_bounds(g);
    if (st0 != FALCON_OK) return st0;
    falcon_comm *cm = g->comm;
    const int P = cm->simulated ? cm->simulated : cm->nranks;
    cudaStream_t s = g->parts[0]->stream;
    std::vector<uint2 *> ho;
    std::vector<uint32_t *> hc;
    for (auto *p : g->parts) {
        CU(dmalloc(&p->xcounts, (size_t)P));
        CU(dmalloc(&p->outbox, (size_t)g->n));
        if (!cm->simulated) {
            CU(dmalloc(&p->xcnt_recv, (size_t)P));
            CU(dmalloc(&p->inbox, (size_t)(p->hi - p->lo) * (size_t)(P > 1 ? P - 1 : 1) + 1));
        }
        ho.push_back(p->outbox);
        hc.push_back(p->xcounts);
    }
    if (cm->simulated) {
        CU(dmalloc(&g->d_outboxes, (size_t)P));
        CU(dmalloc(&g->d_counts, (size_t)P));
        CU(cudaMemcpyAsync(g->d_outboxes, ho.data(), sizeof(uint2 *) * P, cudaMemcpyHostToDevice, s));
        CU(cudaMemcpyAsync(g->d_counts, hc.data(), sizeof(uint32_t *) * P, cudaMemcpyHostToDevice, s));
    }
    CU(cudaStreamSynchronize(s));
    return FALCON_OK;
}

// The rest of a part once its CSR is loaded: owned range, receive buffer of
// the dense exchange, unit-weight arcs (BFS as unit-weight SSSP).
falcon_status_t finish_part(falcon_graph *p, int64_t lo, int64_t hi) {
    p->lo = lo; p->hi = hi;
    CU(dmalloc(&p->recv, (size_t)(hi - lo > 0 ? hi - lo : 1)));
    CU(dmalloc(&p->cw_unit, (size_t)(p->m ? p->m : 1)));
    if (p->m) {
        int32_t *ones = nullptr;
        CU(dmalloc(&ones, (size_t)p->m));
        k_fill_i32<<<p->num_sms * 8, BLOCK, 0, p->stream>>>(ones, (uint64_t)p->m, 1);
        k_interleave<<<p->num_sms * 8, BLOCK, 0, p->stream>>>((uint64_t)p->m, p->col, ones, p->cw_unit);
        CU(cudaStreamSynchronize(p->stream));
        dfree(ones);
    }
    return FALCON_OK;
}

// Build the part owning [lo, hi) from the FULL CSR: its rows only, global ids, full n.
falcon_status_t load_part(int64_t n, const uint32_t *h_row_off, const uint32_t *col, const int32_t *w, int64_t lo,
                          int64_t hi, int device, void *stream, falcon_graph **out) {
    std::vector<uint32_t> ro((size_t)n + 1);
    const uint32_t base = h_row_off[lo], top = h_row_off[hi];
    for (int64_t v = 0; v <= n; v++) {
        const uint32_t r = h_row_off[v < lo ? lo : (v > hi ? hi : v)];
        ro[(size_t)v] = r - base;
    }
    falcon_load_opts_t o = {};
    o.device = device;
    o.cuda_stream = stream;
    falcon_graph *p = new (std::nothrow) falcon_graph();
    if (!p) return fail(FALCON_ERR_NO_MEMORY, "host allocation failed");
    const int64_t mp = (int64_t)(top - base);
    falcon_status_t st = load(n, mp, ro.data(), col + base, w ? w + base : nullptr, &o, p);
    if (st == FALCON_OK) st = finish_part(p, lo, hi);
    if (st != FALCON_OK) { destroy(p); return st; }
    *out = p;
    return FALCON_OK;
}

// Full-length row offsets of a slice part: 0 before lo, the slice's offsets
// on [lo, hi], m_local after hi (rows outside the slice are empty).
__global__ void k_slice_rows(uint32_t N, uint32_t lo, uint32_t hi, uint32_t m_local, const uint32_t *slice_ro,
                             uint32_t *ro) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v <= N; v += stride)
        ro[v] = v < lo ? 0u : (v <= hi ? slice_ro[v - lo] : m_local);
}

// FALCON_LOAD_SLICE: this rank passed only its rows.  The ranks all-gather
// their (rows, arcs) counts; rank r owns the vertices after those of ranks
// < r.  The rank's CSR is validated on the device (load) against the global
// vertex count -- no full-graph host copy or host loop.
falcon_status_t load_slice(int64_t n_local, int64_t m_local, const uint32_t *row_off, const uint32_t *col,
                           const int32_t *w, const falcon_load_opts_t *opts, falcon_graph *g) {
    falcon_comm *cm = opts->comm;
    const int P = cm->nranks;
    NcclApi *nc = cm->api;
    const int device = cm->device;
    CU(cudaSetDevice(device));
    cudaStream_t s = nullptr;
    CU(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct SGuard { cudaStream_t s; ~SGuard() { cudaStreamSynchronize(s); cudaStreamDestroy(s); } } sg{s};
    uint64_t *d_cnt = nullptr;
    CU(dmalloc(&d_cnt, 2 * (size_t)P + 2));
    uint64_t mine[2] = {(uint64_t)n_local, (uint64_t)m_local};
    CU(cudaMemcpyAsync(d_cnt + 2 * P, mine, sizeof mine, cudaMemcpyHostToDevice, s));
    NC(nc->AllGather(d_cnt + 2 * P, d_cnt, 2, ncclUint64, cm->nccl, s));
    std::vector<uint64_t> cnt(2 * (size_t)P);
    CU(cudaMemcpyAsync(cnt.data(), d_cnt, sizeof(uint64_t) * 2 * P, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    dfree(d_cnt);
    uint64_t N = 0, M = 0;
    g->bounds.assign((size_t)P + 1, 0);
    for (int q = 0; q < P; q++) {
        g->bounds[(size_t)q] = (int64_t)N;
        N += cnt[2 * (size_t)q];
        M += cnt[2 * (size_t)q + 1];
    }
    g->bounds[(size_t)P] = (int64_t)N;
    if (N < 1 || N >= (1ull << 31)) return fail(FALCON_ERR_INVALID_ARG, "the slices hold %llu vertices (need [1, 2^31))",
                                                (unsigned long long)N);
    g->n = (int64_t)N; g->m = (int64_t)M;
    const int64_t lo = g->bounds[(size_t)cm->rank], hi = g->bounds[(size_t)cm->rank + 1];
    // the slice's first and last offsets (host or device pointer)
    uint32_t ends[2] = {1, 0};
    CU(cudaMemcpy(&ends[0], row_off, 4, cudaMemcpyDefault));
    CU(cudaMemcpy(&ends[1], row_off + n_local, 4, cudaMemcpyDefault));
    if (ends[0] != 0 || ends[1] != (uint64_t)m_local)
        return fail(FALCON_ERR_OUT_OF_RANGE, "slice row_off must start at 0 and end at m");
    uint32_t *d_slice = nullptr, *d_ro = nullptr;
    CU(dmalloc(&d_slice, (size_t)n_local + 1));
    CU(dmalloc(&d_ro, (size_t)N + 1));
    CU(cudaMemcpyAsync(d_slice, row_off, ((size_t)n_local + 1) * 4, cudaMemcpyDefault, s));
    k_slice_rows<<<1184, BLOCK, 0, s>>>((uint32_t)N, (uint32_t)lo, (uint32_t)hi, (uint32_t)m_local, d_slice, d_ro);
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(s));
    falcon_load_opts_t o = {};
    o.device = device;
    o.cuda_stream = opts->cuda_stream;
    falcon_graph *p = new (std::nothrow) falcon_graph();
    if (!p) return fail(FALCON_ERR_NO_MEMORY, "host allocation failed");
    falcon_status_t st = load((int64_t)N, m_local, d_ro, col, w, &o, p);   // device validation: col < N, w >= 0
    dfree(d_slice);
    dfree(d_ro);
    if (st == FALCON_OK) st = finish_part(p, lo, hi);
    if (st != FALCON_OK) { destroy(p); return st; }
    g->parts.push_back(p);
    return FALCON_OK;
}

falcon_status_t load_partitioned(int64_t n, int64_t m, const uint32_t *row_off, const uint32_t *col, const int32_t *w,
                                 const falcon_load_opts_t *opts, falcon_graph *g) {
    falcon_comm *cm = opts->comm;
    g->comm = cm;
    g->gather = (opts->flags & FALCON_LOAD_GATHER) != 0;
    const int P = cm->simulated ? cm->simulated : cm->nranks;
    if (opts->flags & FALCON_LOAD_SLICE) {
        if (cm->simulated)
            return fail(FALCON_ERR_UNSUPPORTED, "FALCON_LOAD_SLICE needs a rank communicator (one handle per rank)");
        falcon_status_t st = load_slice(n, m, row_off, col, w, opts, g);
        if (st != FALCON_OK) return st;
    } else {
        g->n = n; g->m = m;
        // host copy of the offsets (the caller's may live on the device)
        std::vector<uint32_t> h_ro((size_t)n + 1);
        CU(cudaMemcpy(h_ro.data(), row_off, ((size_t)n + 1) * 4, cudaMemcpyDefault));
        if (h_ro[0] != 0 || h_ro[(size_t)n] != (uint64_t)m)
            return fail(FALCON_ERR_OUT_OF_RANGE, "row_off must start at 0 and end at m");
        for (int64_t v = 0; v < n; v++)
            if (h_ro[(size_t)v] > h_ro[(size_t)v + 1])
                return fail(FALCON_ERR_OUT_OF_RANGE, "row_off must be nondecreasing");
        g->bounds.assign((size_t)P + 1, 0);
        partition_bounds(n, h_ro.data(), P, g->bounds.data());
        const int device = cm->simulated ? (opts->device >= 0 ? opts->device : 0) : cm->device;
        CU(cudaSetDevice(device));
        for (int q = 0; q < P; q++) {
            if (!cm->simulated && q != cm->rank) continue;
            falcon_graph *p = nullptr;
            falcon_status_t st = load_part(n, h_ro.data(), col, w, g->bounds[q], g->bounds[q + 1], device,
                                           opts->cuda_stream, &p);
            if (st != FALCON_OK) return st;
            g->parts.push_back(p);
        }
    }
    g->device = g->parts[0]->device;
    g->lo = cm->simulated ? 0 : g->bounds[cm->rank];
    g->hi = cm->simulated ? g->n : g->bounds[cm->rank + 1];
    g->stream = g->parts[0]->stream;
    if (const char *ex = getenv("FALCON_EXCHANGE")) g->exchange = (uint32_t)atoi(ex) % 4u;
    return FALCON_OK;
}

// Sparse exchange: pack the pairs per owner, move them (device reads when
// simulated; grouped ncclSend / ncclRecv after a count exchange otherwise),
// apply them on the owners with atomicMin.
falcon_status_t exchange_sparse(falcon_graph *g, const std::vector<Args> &args, cudaStream_t s) {
    falcon_comm *cm = g->comm;
    const int P = cm->simulated ? cm->simulated : cm->nranks;
    for (size_t i = 0; i < g->parts.size(); i++) {
        falcon_graph *p = g->parts[i];
        CU(cudaMemsetAsync(p->xcounts, 0, (size_t)P * 4, s));
        k_remote_pairs<true><<<p->grid_small, BLOCK, 0, s>>>(args[i], (uint32_t)p->lo, (uint32_t)p->hi, g->bounds_d, P,
                                                             p->xcounts, p->outbox);
    }
    if (cm->simulated) {
        for (int q = 0; q < P; q++) {
            falcon_graph *p = g->parts[(size_t)q];
            k_sim_apply_pairs<<<p->grid_small, BLOCK, 0, s>>>(args[(size_t)q], g->d_outboxes, g->d_counts, P, q,
                                                              (uint32_t)p->lo);
        }
        k_sum_counts<<<1, 64, 0, s>>>(g->d_counts, P, g->xpairs_d);   // bytes moved, read once per call
        return FALCON_OK;
    }
    NcclApi *nc = cm->api;
    if (!nc->Send || !nc->Recv) return fail(FALCON_ERR_COMM, "ncclSend/ncclRecv unavailable");
    falcon_graph *me = g->parts[0];
    const int r = cm->rank;
    NC(nc->GroupStart());   // counts: what every peer sends to me
    for (int q = 0; q < P; q++) {
        if (q == r) continue;
        NC(nc->Send(me->xcounts + q, 1, ncclUint32, q, cm->nccl, s));
        NC(nc->Recv(me->xcnt_recv + q, 1, ncclUint32, q, cm->nccl, s));
    }
    NC(nc->GroupEnd());
    std::vector<uint32_t> hs((size_t)P), hr((size_t)P);
    CU(cudaMemcpyAsync(hs.data(), me->xcounts, (size_t)P * 4, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(hr.data(), me->xcnt_recv, (size_t)P * 4, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    uint64_t in_total = 0;
    // payloads: my pairs for q from my outbox region q, q's pairs for me into
    // my inbox.  Every pair of ranks exchanges a message, possibly empty, so
    // every rank takes part in the group (the loopback transport matches whole
    // groups; NCCL accepts zero-count sends).
    NC(nc->GroupStart());
    for (int q = 0; q < P; q++) {
        if (q == r) continue;
        NC(nc->Send(me->outbox + g->bounds[(size_t)q], 2 * (size_t)hs[(size_t)q], ncclUint32, q, cm->nccl, s));
        NC(nc->Recv(me->inbox + in_total, 2 * (size_t)hr[(size_t)q], ncclUint32, q, cm->nccl, s));
        in_total += hr[(size_t)q];
        g->xbytes += 8ull * hs[(size_t)q];
    }
    NC(nc->GroupEnd());
    if (in_total) k_apply_pairs<<<me->grid_small, BLOCK, 0, s>>>(args[0], me->inbox, (uint32_t)in_total);
    return FALCON_OK;
}

// Gather the full n-array into dst (device): every part's owned range.
falcon_status_t gather_full(falcon_graph *g, int32_t *dst, cudaStream_t s) {
    falcon_comm *cm = g->comm;
    if (cm->simulated) {
        for (auto *p : g->parts)
            if (p->hi > p->lo)
                CU(cudaMemcpyAsync(dst + p->lo, p->val + p->lo, (size_t)(p->hi - p->lo) * 4, cudaMemcpyDefault, s));
        return FALCON_OK;
    }
    NcclApi *nc = cm->api;
    falcon_graph *me = g->parts[0];
    NC(nc->GroupStart());
    for (int q = 0; q < cm->nranks; q++) {
        const int64_t qlo = g->bounds[(size_t)q], qcnt = g->bounds[(size_t)q + 1] - qlo;
        if (qcnt == 0) continue;
        NC(nc->Broadcast(me->val + qlo, dst + qlo, (size_t)qcnt, ncclInt32, q, cm->nccl, s));
    }
    NC(nc->GroupEnd());
    return FALCON_OK;
}

// One partitioned call.  Output: this rank's owned slice [lo, hi) (NCCL /
// loopback ranks), the full n-array with FALCON_LOAD_GATHER or simulated.
falcon_status_t run_partitioned(falcon_graph *g, int algo, uint32_t source, int32_t *out, falcon_stats_t *stats) {
    if (!out) return fail(FALCON_ERR_INVALID_ARG, "output pointer is NULL");
    if (algo != CC && (int64_t)source >= g->n) return fail(FALCON_ERR_INVALID_ARG, "source %u >= n", source);
    falcon_comm *cm = g->comm;
    const int P = (int)g->parts.size();
    NcclApi *nc = cm->simulated ? nullptr : cm->api;
    if (!cm->simulated && !nc) return fail(FALCON_ERR_COMM, "no communicator transport");
    CU(cudaSetDevice(g->device));
    cudaStream_t s = g->parts[0]->stream;   // simulated parts share the device; order them on one stream
    const uint32_t cap = (uint32_t)(g->n + 2 > 0xFFFFFFF0ll ? 0xFFFFFFF0ll : g->n + 2);
    std::vector<Args> args;
    for (auto *p : g->parts) {
        p->use_unit = algo == BFS;
        args.push_back(p->args());
    }
    // device pointer tables for the simulated exchange
    int32_t **d_vals = nullptr;
    Ctrl **d_ctrls = nullptr;
    if (cm->simulated) {
        std::vector<int32_t *> hv;
        std::vector<Ctrl *> hc;
        for (auto *p : g->parts) { hv.push_back(p->val); hc.push_back(p->ctrl); }
        CU(dmalloc(&d_vals, (size_t)P));
        CU(dmalloc(&d_ctrls, (size_t)P));
        CU(cudaMemcpyAsync(d_vals, hv.data(), sizeof(int32_t *) * P, cudaMemcpyHostToDevice, s));
        CU(cudaMemcpyAsync(d_ctrls, hc.data(), sizeof(Ctrl *) * P, cudaMemcpyHostToDevice, s));
    }
    // exchange mode: 1 dense, 2 sparse, 3 fused; auto (0) = fused between
    // ranks that can map each other's memory, else dense
    uint32_t mode = g->exchange;
    if (algo == CC) mode = 1;
    if (mode == 0) mode = cm->simulated ? 1 : (ensure_fused(g) == FALCON_OK ? 3 : 1);
    const bool fused = mode == 3;
    if (fused) {
        falcon_status_t st = ensure_fused(g);
        if (st != FALCON_OK) return st;
        for (size_t i = 0; i < g->parts.size(); i++) {
            falcon_graph *p = g->parts[i];
            // every part of the communicator (an NCCL rank holds only its own part)
            args[i].lo = (uint32_t)p->lo; args[i].hi = (uint32_t)p->hi;
            args[i].nparts = (uint32_t)(cm->simulated ? cm->simulated : cm->nranks);
            args[i].bounds = g->bounds_d; args[i].peer_val = g->d_peer_val; args[i].peer_bm = g->d_peer_bm;
        }
    }
    g_last_error.clear();
    CU(cudaEventRecord(g->parts[0]->ev0, s));
    g->xbytes = 0;
    if (g->xpairs_d) CU(cudaMemsetAsync(g->xpairs_d, 0, 8, s));
    const int init_algo = algo == CC ? CC : SSSP;
    for (size_t i = 0; i < g->parts.size(); i++) {
        falcon_graph *p = g->parts[i];
        if (init_algo == CC) k_init<CC><<<p->grid_small, BLOCK, 0, s>>>(args[i], 0, cap, 3u * p->cnt_slots, VERTEX, 1);
        else k_init<SSSP><<<p->grid_small, BLOCK, 0, s>>>(args[i], source, cap, 3u * p->cnt_slots, VERTEX, 1);
    }
    CU(cudaGetLastError());
    if (fused && !cm->simulated) {   // every rank's init is complete before any peer writes into it
        NC(nc->AllReduce(&g->parts[0]->ctrl->changed, &g->parts[0]->ctrl->changed, 1, ncclUint32, ncclSum,
                         cm->nccl, s));
    }
    int64_t rounds = 0, host_checks = 0;
    for (;;) {
        for (int k = 0; k < HOST_CHECK_EVERY; k++) {
            rounds++;
            // 1. relax
            for (size_t i = 0; i < g->parts.size(); i++) {
                falcon_graph *p = g->parts[i];
                if (algo == CC) {
                    launch_l2(p, k_cc_vertex<BLOCK>, p->grid_cc, s, args[i]);
                } else if (fused) {   // remote targets land in their owners' arrays: no exchange step
                    launch_l2(p, k_expand_warp<SSSP, VFUSED, BLOCK, 4, 3>, p->grid_expand_fr, s, args[i]);
                } else {
                    launch_expand_warp<SSSP, VERTEX>(p, s, args[i]);
                }
            }
            // 2.-3. exchange + apply
            if (algo == CC) {
                if (cm->simulated) {
                    k_sim_allreduce_min<<<g->parts[0]->grid_small, BLOCK, 0, s>>>(d_vals, P, (uint32_t)g->n);
                } else {
                    NC(nc->AllReduce(g->parts[0]->val, g->parts[0]->val, (size_t)g->n, ncclInt32, ncclMin, cm->nccl, s));
                    g->xbytes += 4ull * (uint64_t)g->n;
                }
                for (size_t i = 0; i < g->parts.size(); i++)
                    launch_l2(g->parts[i], k_compress, g->parts[i]->grid_small, s, args[i]);
            } else if (fused) {
                // nothing to exchange: the relax kernels wrote into the owners
            } else {
                const int NP = cm->simulated ? P : cm->nranks;
                const bool sparse = mode == 2 && NP > 1;
                if (sparse) {
                    falcon_status_t st = ensure_sparse(g);
                    if (st != FALCON_OK) return st;
                }
                if (sparse) {
                    falcon_status_t st = exchange_sparse(g, args, s);
                    if (st != FALCON_OK) return st;
                } else if (cm->simulated) {
                    g->xbytes += 4ull * (uint64_t)g->n * (uint64_t)(P - 1);
                    for (int q = 0; q < P; q++) {
                        falcon_graph *p = g->parts[(size_t)q];
                        k_sim_reduce_min<<<p->grid_small, BLOCK, 0, s>>>(d_vals, P, (uint32_t)p->lo,
                                                                           (uint32_t)(p->hi - p->lo), p->recv);
                    }
                } else {
                    g->xbytes += 4ull * (uint64_t)(g->n - (g->hi - g->lo));
                    falcon_graph *me = g->parts[0];
                    NC(nc->GroupStart());
                    for (int q = 0; q < cm->nranks; q++) {
                        const int64_t qlo = g->bounds[(size_t)q], qcnt = g->bounds[(size_t)q + 1] - qlo;
                        if (qcnt == 0) continue;
                        NC(nc->Reduce(me->val + qlo, me->recv, (size_t)qcnt, ncclInt32, ncclMin, q, cm->nccl, s));
                    }
                    NC(nc->GroupEnd());
                }
                for (size_t i = 0; i < g->parts.size() && !sparse; i++) {
                    falcon_graph *p = g->parts[i];
                    if (p->hi > p->lo)
                        k_apply_owned<<<p->grid_small, BLOCK, 0, s>>>(args[i], p->recv, (uint32_t)p->lo,
                                                                      (uint32_t)(p->hi - p->lo));
                }
            }
            // 4. termination: every part sees the global `changed`
            if (cm->simulated) {
                k_sim_sum_changed<<<1, 32, 0, s>>>(d_ctrls, P);
            } else {
                NC(nc->AllReduce(&g->parts[0]->ctrl->changed, &g->parts[0]->ctrl->changed, 1, ncclUint32, ncclSum,
                                 cm->nccl, s));
            }
            for (size_t i = 0; i < g->parts.size(); i++) {
                if (algo == CC)
                    k_advance<CC, VERTEX><<<1, 32, 0, s>>>(g->parts[i]->ctrl, 0, 0, 0u, (uint32_t)g->n, 0u, 0u, 0u, 0u, 0u);
                else
                    k_advance<SSSP, VERTEX><<<1, 32, 0, s>>>(g->parts[i]->ctrl, 0, 0, 0u, (uint32_t)g->n, 0u, 0u, 0u, 0u, 0u);
            }
        }
        CU(cudaGetLastError());
        host_checks++;   // the only host round trip: once per HOST_CHECK_EVERY supersteps
        CU(cudaMemcpyAsync(g->parts[0]->h_ctrl, g->parts[0]->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        if (g->parts[0]->h_ctrl->done) break;
    }
    for (size_t i = 0; i < g->parts.size(); i++)
        k_finish<<<1, BLOCK, 0, s>>>(args[i], (uint32_t)g->parts[i]->cnt_slots);
    if (cm->simulated && g->xpairs_d) {
        unsigned long long pairs = 0;
        CU(cudaMemcpyAsync(&pairs, g->xpairs_d, 8, cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        g->xbytes += 8ull * pairs;
    }
    // output: the owned slice, or the full array on every rank
    const bool full_out = cm->simulated || g->gather;
    cudaPointerAttributes at;
    const bool out_on_device = cudaPointerGetAttributes(&at, out) == cudaSuccess &&
                               (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged);
    cudaGetLastError();
    int32_t *full = nullptr, *staging = nullptr;
    if (full_out) {
        if (!out_on_device) CU(dmalloc(&staging, (size_t)g->n));
        full = out_on_device ? out : staging;
        falcon_status_t st = gather_full(g, full, s);
        if (st != FALCON_OK) return st;
    }
    CU(cudaEventRecord(g->parts[0]->ev1, s));
    if (full_out) {
        if (staging) CU(cudaMemcpyAsync(out, staging, (size_t)g->n * 4, cudaMemcpyDeviceToHost, s));
    } else if (g->hi > g->lo) {
        CU(cudaMemcpyAsync(out, g->parts[0]->val + g->lo, (size_t)(g->hi - g->lo) * 4, cudaMemcpyDefault, s));
    }
    std::vector<Ctrl> hc(g->parts.size());
    for (size_t i = 0; i < g->parts.size(); i++)
        CU(cudaMemcpyAsync(&hc[i], g->parts[i]->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    if (fused)   // each remote improvement moved a RED.MIN (4 B) and a bitmap RED.OR (4 B) to its owner
        for (auto &c : hc) g->xbytes += 8ull * c.xremote;
    bool overflow = false;
    {   // overflow certificate (R3) over every part's rows against the full array
        uint32_t any = 0;
        for (auto &c : hc) any |= c.cand_ovf;
        falcon_graph *me = g->parts[0];
        if (!cm->simulated) {   // the same decision on every rank
            CU(cudaMemcpyAsync(me->d_flags, &any, 4, cudaMemcpyHostToDevice, s));
            NC(nc->AllReduce(me->d_flags, me->d_flags, 1, ncclUint32, ncclMax, cm->nccl, s));
            CU(cudaMemcpyAsync(&any, me->d_flags, 4, cudaMemcpyDeviceToHost, s));
            CU(cudaStreamSynchronize(s));
        }
        if (algo == SSSP && any) {
            int32_t *arr = full;
            int32_t *tmp = nullptr;
            if (!arr) {   // owned-slice output: gather a full copy for the certificate (rare path)
                CU(dmalloc(&tmp, (size_t)g->n));
                falcon_status_t st = gather_full(g, tmp, s);
                if (st != FALCON_OK) return st;
                CU(cudaStreamSynchronize(s));
                arr = tmp;
            }
            int flag = 0;
            for (auto *p : g->parts) {
                bool bad = false;
                falcon_status_t st = overflow_certificate(p, p->row_off, p->col, arr, &bad);
                if (st != FALCON_OK) return st;
                flag |= bad ? 1 : 0;
            }
            dfree(tmp);
            if (!cm->simulated) {
                CU(cudaMemcpyAsync(me->d_flags, &flag, 4, cudaMemcpyHostToDevice, s));
                NC(nc->AllReduce(me->d_flags, me->d_flags, 1, ncclInt32, ncclMax, cm->nccl, s));
                CU(cudaMemcpyAsync(&flag, me->d_flags, 4, cudaMemcpyDeviceToHost, s));
                CU(cudaStreamSynchronize(s));
            }
            overflow = flag != 0;
        }
    }
    dfree(staging);
    dfree(d_vals);
    dfree(d_ctrls);
    for (auto *p : g->parts) p->use_unit = false;
    g->last_mode = mode;
    g->last_rounds = rounds;
    g->last_host_checks = host_checks;
    if (stats) {
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, g->parts[0]->ev0, g->parts[0]->ev1));
        memset(stats, 0, sizeof *stats);
        stats->iterations = hc[0].iter;
        for (auto &c : hc) {
            stats->vertices_processed += (int64_t)c.vertices;
            stats->edges_relaxed += (int64_t)c.edges;
            stats->updates += (int64_t)c.updates;
        }
        stats->kernel_launches = rounds * (algo == CC ? 3 : (fused ? 2 : 3)) * (int64_t)g->parts.size() + 2;
        stats->ms = ms;
        stats->relax_ms = -1.0;
    }
    for (auto &c : hc)
        if (c.status == ST_NOT_CONVERGED) return fail(FALCON_ERR_NOT_CONVERGED, "no fixpoint within %u rounds", cap);
    for (auto &c : hc)
        if (c.status == ST_QUEUE) return fail(FALCON_ERR_CUDA, "internal error: frontier queue bound exceeded");
    if (overflow) return fail(FALCON_ERR_OVERFLOW, "a finite shortest distance is >= FALCON_INF");
    g_last_error.clear();
    return FALCON_OK;
}

}  // namespace
