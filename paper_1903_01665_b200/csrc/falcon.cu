// falcon.cu -- C ABI (include/falcon.h), device graph store and the
// single-GPU fixpoint driver.
//
// Driver: one fused init kernel, then a CUDA graph whose WHILE
// conditional node runs one round per trip -- relax kernel(s) followed by a
// one-thread advance kernel that decides on the device whether to continue
// (cudaGraphSetConditional).  No host round trip per round, unlike the
// per-iteration `changed` copy of the paper's generated code (PAPER.md:1595,
// 1682-1684).  The graphs are built once per (graph, algorithm,
// style) and cached.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: one named range per C-ABI call (no link dependency)

#include <atomic>
#include <cstdarg>
#include <map>
#include <mutex>
#include <unordered_map>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>
#include <utility>
#include <vector>

#include "../../include/falcon.h"
#include "kernels.cuh"
#include "cc.cuh"
#include "mst.cuh"

using namespace fk;

namespace {

constexpr int BLOCK = 256;
constexpr int UNROLL = 4;   // arcs per thread per expansion step
// EDGE style: 4-arc quads per lane per warp chunk, per algorithm (measured on
// B200: SSSP prefers short chunks -- 48 registers, 5 CTAs/SM; BFS longer ones)
constexpr int EDGE_QP_SSSP = 1, EDGE_QP_BFS = 2;
constexpr uint32_t ECH_SSSP = 128u * EDGE_QP_SSSP, ECH_BFS = 128u * EDGE_QP_BFS;   // arcs per warp chunk
constexpr int HOST_CHECK_EVERY = 4;
constexpr uint64_t MAX_BLOCKS_USED = 4;   // destination blocks of the SSSP layout (<= MAX_BLK)

thread_local std::string g_last_error;

falcon_status_t fail(falcon_status_t st, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return st;
}

#define CU(call)                                                                                      \
    do {                                                                                              \
        cudaError_t _e = (call);                                                                      \
        if (_e != cudaSuccess) {                                                                      \
            if (_e == cudaErrorMemoryAllocation)                                                      \
                return fail(FALCON_ERR_NO_MEMORY, "%s: %s", #call, cudaGetErrorString(_e));           \
            return fail(FALCON_ERR_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(_e)); \
        }                                                                                             \
    } while (0)

// Device memory: a per-process caching allocator over cudaMalloc.  A freed
// block (graph_free, per-call staging buffers) goes back to a cache keyed by
// (device, size class) instead of to cudaFree -- which synchronises the device
// and unmaps, ~7 ms for one rand-25M graph -- and the next allocation of that
// class reuses it (the next graph of the same shape, the next call's
// staging).  Size classes: 256 B below 1 MiB, 2 MiB above.  When cudaMalloc
// fails the device's cached blocks are released and the allocation retried.
// Callers free a block only after the work that uses it has completed.
struct DevCache {
    std::mutex mu;
    std::multimap<std::pair<int, size_t>, void *> idle;    // (device, bytes) -> block
    std::unordered_map<void *, std::pair<int, size_t>> live;
};
DevCache &dev_cache() {
    static DevCache *c = new DevCache();   // never destroyed: blocks may be freed during process exit
    return *c;
}

cudaError_t dev_alloc(void **p, size_t bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    const size_t gran = bytes < (1u << 20) ? 256 : (2u << 20);
    bytes = (bytes + gran - 1) / gran * gran;
    DevCache &c = dev_cache();
    {
        std::lock_guard<std::mutex> lk(c.mu);
        auto it = c.idle.find({dev, bytes});
        if (it != c.idle.end()) {
            *p = it->second;
            c.idle.erase(it);
            c.live[*p] = {dev, bytes};
            return cudaSuccess;
        }
    }
    cudaError_t e = cudaMalloc(p, bytes);   // 256-byte aligned: the 16-byte vector loads rely on it
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        std::vector<void *> rel;
        {
            std::lock_guard<std::mutex> lk(c.mu);
            for (auto it = c.idle.begin(); it != c.idle.end();) {
                if (it->first.first == dev) { rel.push_back(it->second); it = c.idle.erase(it); }
                else ++it;
            }
        }
        for (void *q : rel) cudaFree(q);
        e = cudaMalloc(p, bytes);
    }
    if (e == cudaSuccess) {
        std::lock_guard<std::mutex> lk(c.mu);
        c.live[*p] = {dev, bytes};
    }
    return e;
}

void dfree(void *p) {
    if (!p) return;
    DevCache &c = dev_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.live.find(p);
    if (it == c.live.end()) return;
    c.idle.insert({it->second, p});
    c.live.erase(it);
}

// Pinned host copies of the control block: recycled through a free list, as
// cudaFreeHost unregisters the page and can take tens to hundreds of ms on a
// busy host (measured 16-515 ms per graph_free on this pool's boxes).
struct HostCtrlCache {
    std::mutex mu;
    std::vector<void *> idle;
};
HostCtrlCache &host_ctrl_cache() {
    static HostCtrlCache *c = new HostCtrlCache();
    return *c;
}
cudaError_t host_ctrl_alloc(void **p, size_t bytes) {
    HostCtrlCache &c = host_ctrl_cache();
    {
        std::lock_guard<std::mutex> lk(c.mu);
        if (!c.idle.empty()) { *p = c.idle.back(); c.idle.pop_back(); return cudaSuccess; }
    }
    return cudaMallocHost(p, bytes < 4096 ? 4096 : bytes);
}
void host_ctrl_free(void *p) {
    if (!p) return;
    HostCtrlCache &c = host_ctrl_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    c.idle.push_back(p);
}

template <typename T>
cudaError_t dmalloc(T **p, size_t count) {
    return dev_alloc(reinterpret_cast<void **>(p), (count ? count : 1) * sizeof(T));
}

}  // namespace

// NVTX range for the duration of one C-ABI call (visible in nsys / ncu --nvtx).
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
const char *const NVTX_SSSP[4] = {"falcon_sssp VERTEX", "falcon_sssp EDGE", "falcon_sssp WORKLIST", "falcon_sssp DELTA"};
const char *const NVTX_BFS[4] = {"falcon_bfs VERTEX", "falcon_bfs EDGE", "falcon_bfs WORKLIST", "falcon_bfs ?"};
const char *const NVTX_CC[4] = {"falcon_cc VERTEX", "falcon_cc EDGE", "falcon_cc WORKLIST", "falcon_cc ?"};

struct falcon_graph {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    cudaStream_t cap_stream = nullptr;
    int64_t n = 0, m = 0;
    uint32_t *row_off = nullptr, *col = nullptr, *src = nullptr;
    int32_t *w = nullptr;
    uint2 *cw = nullptr;
    uint32_t *rowb = nullptr, *srcb = nullptr;   // destination-blocked layout (SSSP), built lazily
    uint2 *cwb = nullptr;
    uint2 *chunk = nullptr, *chunkb = nullptr;   // EDGE chunk source ranges: of src (BFS chunks) / srcb (SSSP chunks)
    uint2 *chunks = nullptr;                     // ... of src in SSSP chunks (unblocked graphs)
    uint32_t nblk = 1, bsz = 0;
    size_t blk_bytes = 64u << 20;        // value-array bytes per block (FALCON_BLOCK_MB)
    uint32_t dense_div = 32;             // dense round: frontier > n / dense_div (FALCON_DENSE_DIV; swept 8-128)
    uint32_t blk_div = 8;                // blocked round: frontier > n / blk_div (FALCON_BLOCK_DIV)
    uint32_t wl_noq = 1;                 // WORKLIST dense rounds without claims / queue (FALCON_WL_NOQ)
    uint32_t dl_noq = 1;                 // ... DELTA dense rounds (FALCON_DL_NOQ)
    // SSSP DELTA sparse rounds: local continuation tiles per warp, in rounds of
    // at most local_max items (FALCON_LOCAL / FALCON_LOCAL_MAX; set at load:
    // 16 / unbounded on sparse high-diameter graphs (m < 3n), 4 / 16384 below
    // m = 6n, else off --
    // tools/survey.py sweep, profiles/r01_local.log)
    uint32_t local_tiles = 4;
    uint32_t local_max = 16384;
    // ... SSSP WORKLIST (FALCON_WL_LOCAL / FALCON_WL_LOCAL_MAX; set at load:
    // 4 tiles in rounds of <= 256 K items when m < 3n, else off)
    uint32_t wl_local_tiles = 0;
    uint32_t wl_local_max = 262144;
    uint32_t delta_cap = 0;              // adaptive Δ growth cap x Δ0 (0 = 128; FALCON_DELTA_CAP)
    int32_t bfs_unit = -1;               // BFS WORKLIST as unit-weight Δ-stepping: -1 auto (m < 3n), 0 off, 1 on
    bool unit_run = false;               // the call in flight is such a BFS: arcs from cw_unit
    uint32_t *rin_off = nullptr, *rin_col = nullptr;   // reverse CSR (BFS pull), built lazily
    uint32_t lazy_div = 256;             // BFS VERTEX lazy visited set in push rounds with frontier > n / lazy_div
                                         // (option bfs_lazy_div / FALCON_BFS_LAZY_DIV; 0 = never)
    uint32_t cta_thr = 1024;             // CTA-level expansion of rows longer than this (FALCON_CTA_THR / option cta_thr; 0 = off)
    uint32_t wl_pull = 1;                // BFS WORKLIST: bottom-up rounds like VERTEX (FALCON_BFS_WL_PULL / option
                                         // bfs_wl_pull; 0 = push only)
    uint32_t skip_now = 1;               // SSSP: an item already re-activated for the next round is not expanded now
                                         // (FALCON_SKIP_NOW / option skip_now; 0 = off)
    uint32_t pull_rule = 0;              // BFS VERTEX direction: 0 cost model; 1 / 2 pull iff frontier > n / pull_div,
                                         // word / compacted pull form (FALCON_BFS_PULL_RULE / option pull_rule)
    uint32_t pull_div = 16;              // BFS VERTEX: bottom-up when next frontier > n / pull_div (0 = never)
    uint32_t split_div = 0;              // DELTA (auto Δ): halve the bucket when a near round hands on > n / split_div
                                         // items (FALCON_SPLIT_DIV; 0 = never)
    int32_t *val = nullptr;
    uint8_t *lv8 = nullptr;              // BFS byte levels (kernels.cuh put_level)
    uint32_t *bm = nullptr, *fr0 = nullptr, *fr1 = nullptr;   // bm: 4 bitmaps of nwords
    uint32_t *tiles = nullptr;           // scan tile sums (load-time layout builds)
    uint32_t nwords = 0;
    Ctrl *ctrl = nullptr;
    Ctrl *h_ctrl = nullptr;
    unsigned long long *cnt = nullptr;
    int *d_flags = nullptr;
    int num_sms = 0;
    int grid_persist = 0, grid_expand_fr = 0, grid_expand_dl = 0, grid_pull = 0, grid_cc = 0, grid_edge = 0, grid_edge_b = 0, grid_small = 0, cnt_slots = 0;
    cudaGraph_t graphs[3][4] = {};
    cudaGraphExec_t execs[3][4] = {};
    int32_t delta = 0;                   // DELTA bucket width (0 = auto: max(1, average weight))
    int32_t delta_auto = 0;
    bool profiling = false;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::vector<cudaEvent_t> pev;
    int variant = 0;                     // FALCON_EXPAND_VARIANT
    bool persist = false;                // queue styles: small rounds in one cooperative kernel (FALCON_PERSIST=1: on)
    uint32_t persist_max = 65536;        // ... while the frontier has at most this many items (FALCON_PERSIST_MAX)
    bool l2_window = false;              // persisting L2 access-policy window on val[]
    cudaAccessPolicyWindow apw = {};

    unsigned long long *mst_best = nullptr;   // MST: per-component best arc key, built lazily
    uint32_t *mst_list = nullptr;             // MST: two live lists (arcs or vertices) of mst_lcap entries
    size_t mst_lcap = 0;
    // ---- views (graph_share): the parent's read-only arrays, own scratch ----
    falcon_graph *parent = nullptr;       // non-NULL: this handle is a view of `parent`
    std::atomic<int> nviews{0};           // (parent) live views (graph_share / graph_free may run on other threads)
    std::mutex unit_mu;                   // (root) guards the lazy build / publication of cw_unit
    // ---- a launched call not yet finished (run_launch / run_finish) ----
    int pend_algo = -1;
    int32_t *pend_out = nullptr;          // pageable host output, copied by run_finish
    uint32_t pend_cap = 0;
    double pend_relax_ms = -1.0;
    int64_t pend_relax_launches = 0, pend_cc_passes = 0, pend_cc_launches = 0;

    // ---- 1-D vertex partition (multi-GPU) ----
    falcon_comm *comm = nullptr;          // non-NULL: this handle is a partitioned graph
    std::vector<falcon_graph *> parts;    // NCCL: this rank's part; simulated: every part
    std::vector<int64_t> bounds;          // part q owns vertices [bounds[q], bounds[q+1])
    int64_t lo = 0, hi = 0;               // (part) owned vertex range
    int32_t *recv = nullptr;              // (part) owned-range receive buffer of the exchange
    uint2 *cw_unit = nullptr;             // (part) unit-weight (col, 1) arcs: BFS as unit-weight SSSP
    bool use_unit = false;
    // sparse exchange (partition.cuh): (part) per-owner counts, outbox of (vertex,
    // value) pairs in per-owner regions, NCCL inbox; (partitioned handle)
    // device copies of the bounds and, simulated, tables of every part's buffers
    uint32_t *xcounts = nullptr, *xcnt_recv = nullptr;
    uint2 *outbox = nullptr, *inbox = nullptr;
    uint32_t *bounds_d = nullptr;
    unsigned long long *xpairs_d = nullptr;   // (simulated) pairs packed by sparse rounds of the current call
    uint2 **d_outboxes = nullptr;
    uint32_t **d_counts = nullptr;
    uint32_t exchange = 0;                // 0 auto, 1 dense, 2 sparse, 3 fused (FALCON_EXCHANGE / option "exchange")
    bool gather = false;                  // (partitioned) FALCON_LOAD_GATHER: full output on every rank
    uint32_t last_mode = 0;               // (partitioned) exchange mode of the last call (1 dense, 2 sparse, 3 fused)
    int64_t last_rounds = 0, last_host_checks = 0;   // (partitioned) supersteps / host round trips of the last call
    int32_t **d_peer_val = nullptr;       // (partitioned, fused) every part's value array / bitmaps
    uint32_t **d_peer_bm = nullptr;
    std::vector<void *> ipc_opened;       // (NCCL, fused) peer mappings to close
    uint64_t xbytes = 0;                  // bytes moved by the exchanges of the last call (all ranks' share here)

    Args args() const {
        Args a{};
        a.n = (uint32_t)n; a.m = (uint32_t)m; a.nwords = nwords;
        a.row_off = row_off; a.col = col; a.w = w; a.cw = use_unit || unit_run ? cw_unit : cw; a.src = src;
        a.rin_off = rin_off; a.rin_col = rin_col;
        const bool blk = rowb && !use_unit && !unit_run;
        a.nblk = blk ? nblk : 1u;
        a.rowb = blk ? rowb : row_off;
        a.cwb = blk ? cwb : a.cw;
        a.srcb = blk ? srcb : src;
        a.chunk = chunk;
        a.chunkb = blk ? chunkb : chunks;
        a.dense_div = dense_div;
        a.blk_div = blk_div;
        a.wl_noq = wl_noq;
        a.dl_noq = dl_noq;
        a.cta_thr = cta_thr;
        a.skip_now = skip_now;
        a.wl_pull = wl_pull && pull_div && !unit_run && rin_off && !persist ? 1u : 0u;
        a.local_tiles = local_tiles;
        a.local_max = local_max;
        a.wl_local_tiles = wl_local_tiles;
        a.wl_local_max = wl_local_max;
        a.delta_cap = delta_cap;
        a.delta_adapt = delta == 0 || unit_run ? 1u : 0u;   // auto Δ adapts per bucket; an explicit Δ is kept
        a.val = val; a.lv8 = lv8; a.fr0 = fr0; a.fr1 = fr1;
        a.bm0 = bm; a.bm1 = bm + nwords; a.bm2 = bm + 2 * (size_t)nwords; a.vis = bm + 3 * (size_t)nwords;
        a.ctrl = ctrl; a.cnt = cnt;
        return a;
    }
};

namespace {

// Launch a relax-round kernel with the graph's L2 access-policy window (the
// gathered value array is marked persisting so the streamed CSR/COO arrays do
// not evict it).  Inside stream capture the attribute becomes
// a kernel-node attribute.
template <typename... KArgs, typename... Act>
void launch_l2(const falcon_graph *g, void (*k)(KArgs...), int grid, cudaStream_t s, Act &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(BLOCK);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    if (g->l2_window) {
        at[0].id = cudaLaunchAttributeAccessPolicyWindow;
        at[0].val.accessPolicyWindow = g->apw;
        cfg.attrs = at;
        cfg.numAttrs = 1;
    }
    cudaLaunchKernelEx(&cfg, k, std::forward<Act>(args)...);
}

// Profiling / tracing: an event after every launch of a round (host-driven
// loop only).  Kinds: 0 = relax kernel (scan, expand, edge), 1 = other.
struct Tracer {
    falcon_graph *g;
    size_t next = 0;
    struct Mark { cudaEvent_t ev; const char *name; int kind; uint32_t round; };
    std::vector<Mark> marks;
    uint32_t round = 0;
    void mark(cudaStream_t s, const char *name, int kind);
};

// Expansion-kernel variants (arcs per lane per step U, min resident CTAs per
// SM): selected at load time by FALCON_EXPAND_VARIANT (tuning experiments).
// Cooperative launch (all CTAs co-resident: the persistent kernel's grid
// barrier relies on it), with the same L2 access-policy window.
template <typename... KArgs, typename... Act>
cudaError_t launch_coop(const falcon_graph *g, void (*k)(KArgs...), int grid, cudaStream_t s, Act &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(BLOCK);
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    int na = 0;
    at[na].id = cudaLaunchAttributeCooperative;
    at[na].val.cooperative = 1;
    na++;
    if (g->l2_window) {
        at[na].id = cudaLaunchAttributeAccessPolicyWindow;
        at[na].val.accessPolicyWindow = g->apw;
        na++;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, k, std::forward<Act>(args)...);
}

template <int ALGO, int STYLE>
void launch_expand_warp(const falcon_graph *g, cudaStream_t s, const Args &a) {
    switch (g->variant) {
    case 1: launch_l2(g, k_expand_warp<ALGO, STYLE, BLOCK, 2, 4>, g->grid_expand_fr, s, a); break;
    case 2: launch_l2(g, k_expand_warp<ALGO, STYLE, BLOCK, 4, 3>, g->grid_expand_fr, s, a); break;
    case 3: launch_l2(g, k_expand_warp<ALGO, STYLE, BLOCK, 2, 6>, g->grid_expand_fr, s, a); break;
    case 4: launch_l2(g, k_expand_warp<ALGO, STYLE, BLOCK, 8, 2>, g->grid_expand_fr, s, a); break;
    case 5: launch_l2(g, k_expand_warp<ALGO, STYLE, BLOCK, 4, 4>, g->grid_expand_dl, s, a); break;
    case 6: launch_l2(g, k_expand_warp<ALGO, STYLE, BLOCK, 3, 4>, g->grid_expand_dl, s, a); break;
    default:   // tuned per style (tools/survey.py sweeps on rand-25M / rmat-10M)
        // DELTA: U = 4 / 3 CTAs per SM where rounds are heavy (rand-25M 3.38 -> 3.08 ms,
        // rmat-10M 4.39 -> 3.14 ms against U = 2 / 4 CTAs), U = 2 / 4 CTAs on sparse
        // high-diameter graphs, whose small local-continuation rounds want the warps
        // (grid-24M 41 ms against 66 ms with U = 4)
        // BFS VERTEX: U = 4 fits 64 registers without spills: 4 CTAs per SM
        // (rand-25M 1.011 -> 0.981 ms; SSSP spills at that bound)
        if (STYLE == DELTA && g->m < 3 * g->n)
            launch_l2(g, k_expand_warp<ALGO, STYLE, BLOCK, 2, 4>, g->grid_expand_dl, s, a);
        else if (ALGO == BFS && STYLE == VERTEX)
            launch_l2(g, k_expand_warp<ALGO, STYLE, BLOCK, 4, 4>, g->grid_expand_dl, s, a);
        else
            launch_l2(g, k_expand_warp<ALGO, STYLE, BLOCK, 4, 3>, g->grid_expand_fr, s, a);
        break;
    }
}

template <int ALGO, int STYLE>
struct Round {
    // Launch one round's kernels on `s`.  Returns the number of launches.
    static int launch(falcon_graph *g, cudaStream_t s, cudaGraphConditionalHandle h, int in_graph, Tracer *tr) {
        Args a = g->args();
        int launches = 0;
        if (tr) tr->mark(s, "begin", 1);
        if (STYLE == VERTEX) {
            if (ALGO == BFS) {
                launch_l2(g, k_pull<BLOCK>, g->grid_pull, s, a);
                launches++;
                if (tr) tr->mark(s, "pull", 0);
            }
            launch_expand_warp<ALGO, VERTEX>(g, s, a);
            if (tr) tr->mark(s, "expand", 0);
        } else if (STYLE == DELTA) {
            if (g->persist) {   // small rounds inside one cooperative kernel
                launch_coop(g, k_persist<SSSP, DELTA, BLOCK, UNROLL>, g->grid_persist, s, a, g->split_div, g->persist_max);
                launches++;
            }
            // the far-set refill (MODE_SCAN rounds) runs inside the expansion kernel
            launch_expand_warp<ALGO, DELTA>(g, s, a);
            if (tr) tr->mark(s, "expand", 0);
        } else if (STYLE == WORKLIST) {
            if (g->persist) {
                launch_coop(g, k_persist<ALGO, WORKLIST, BLOCK, UNROLL>, g->grid_persist, s, a, g->pull_div,
                            g->persist_max);
                launches++;
                if (tr) tr->mark(s, "persist", 0);
            }
            if (ALGO == BFS && a.wl_pull && !g->persist) {   // bottom-up rounds
                launch_l2(g, k_pull<BLOCK>, g->grid_pull, s, a);
                launches++;
                if (tr) tr->mark(s, "pull", 0);
            }
            launch_expand_warp<ALGO, WORKLIST>(g, s, a);
            if (tr) tr->mark(s, "expand", 0);
        } else {
            if (ALGO == SSSP) launch_l2(g, k_edge<SSSP, BLOCK, EDGE_QP_SSSP>, g->grid_edge, s, a);
            else launch_l2(g, k_edge<BFS, BLOCK, EDGE_QP_BFS>, g->grid_edge_b, s, a);
            if (tr) tr->mark(s, "edge", 0);
        }
        launches++;
        launches++;
        k_advance<ALGO, STYLE><<<1, 32, 0, s>>>(g->ctrl, h, in_graph, (uint32_t)launches, (uint32_t)g->n,
                                                 STYLE == DELTA ? g->split_div
                                                 : (STYLE == WORKLIST && !a.wl_pull ? 0u : g->pull_div),
                                                 g->blk_div, g->pull_rule,
                                                 (uint32_t)g->m, g->lazy_div);
        if (tr) tr->mark(s, "advance", 1);
        return launches;
    }
};

void Tracer::mark(cudaStream_t s, const char *name, int kind) {
    while (g->pev.size() <= next) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        g->pev.push_back(e);
    }
    cudaEvent_t e = g->pev[next++];
    cudaEventRecord(e, s);
    marks.push_back({e, name, kind, round});
}

int launch_round(falcon_graph *g, int algo, int style, cudaStream_t s, cudaGraphConditionalHandle h, int in_graph,
                 Tracer *tr) {
#define R(A, S) \
    if (algo == A && style == S) return Round<A, S>::launch(g, s, h, in_graph, tr);
    R(SSSP, VERTEX) R(SSSP, EDGE) R(SSSP, WORKLIST) R(SSSP, DELTA)
    R(BFS, VERTEX) R(BFS, EDGE) R(BFS, WORKLIST)
#undef R
    if (algo == BFS && style == DELTA) return Round<SSSP, DELTA>::launch(g, s, h, in_graph, tr);   // unit-weight BFS
    return 0;
}

falcon_status_t build_graph(falcon_graph *g, int algo, int style) {
    if (g->execs[algo][style]) return FALCON_OK;
    cudaGraph_t G;
    CU(cudaGraphCreate(&G, 0));
    cudaGraphConditionalHandle h;
    CU(cudaGraphConditionalHandleCreate(&h, G, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    CU(cudaGraphAddNode(&node, G, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    CU(cudaStreamBeginCaptureToGraph(g->cap_stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    launch_round(g, algo, style, g->cap_stream, h, 1, nullptr);
    cudaGraph_t captured;
    cudaError_t e = cudaStreamEndCapture(g->cap_stream, &captured);
    if (e != cudaSuccess) {
        cudaGraphDestroy(G);
        return fail(FALCON_ERR_CUDA, "stream capture of the round body failed: %s", cudaGetErrorString(e));
    }
    cudaGraphExec_t X;
    e = cudaGraphInstantiate(&X, G, 0);
    if (e != cudaSuccess) {
        cudaGraphDestroy(G);
        return fail(FALCON_ERR_CUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(e));
    }
    g->graphs[algo][style] = G;
    g->execs[algo][style] = X;
    return FALCON_OK;
}

falcon_status_t ensure_src(falcon_graph *g) {
    if (g->src) return FALCON_OK;
    if (g->m == 0) {
        CU(dmalloc(&g->src, 4));
        return FALCON_OK;
    }
    // built into locals and published only once complete: a failed build
    // leaves the graph without the layout (the next call retries), never
    // with a half-built one (falcon.h: the graph stays valid after an error)
    uint32_t *src = nullptr;
    uint2 *chunk = nullptr, *chunks = nullptr;
    auto undo = [&] { dfree(src); dfree(chunk); dfree(chunks); };
    if (dmalloc(&src, (size_t)g->m) != cudaSuccess ||
        dmalloc(&chunk, (size_t)((g->m + ECH_BFS - 1) / ECH_BFS)) != cudaSuccess ||
        dmalloc(&chunks, (size_t)((g->m + ECH_SSSP - 1) / ECH_SSSP)) != cudaSuccess) {
        undo();
        return fail(FALCON_ERR_NO_MEMORY, "COO sources: device allocation failed");
    }
    k_build_src<<<g->num_sms * 8, BLOCK, 0, g->stream>>>((uint32_t)g->n, (uint32_t)g->m, g->row_off, src);
    k_chunk_range<<<g->num_sms * 8, BLOCK, 0, g->stream>>>((uint32_t)g->m, ECH_BFS, src, chunk);
    k_chunk_range<<<g->num_sms * 8, BLOCK, 0, g->stream>>>((uint32_t)g->m, ECH_SSSP, src, chunks);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
    if (e != cudaSuccess) {
        undo();
        return fail(FALCON_ERR_CUDA, "COO sources: %s", cudaGetErrorString(e));
    }
    g->src = src; g->chunk = chunk; g->chunks = chunks;
    return FALCON_OK;
}

// Destination-blocked copy of the arcs for SSSP, built once
// on the device: nblk = ceil(4n / blk_bytes) blocks (1 = not needed).
falcon_status_t ensure_blocked(falcon_graph *g) {
    if (g->rowb || g->m == 0) return FALCON_OK;
    {
        falcon_status_t st = ensure_src(g);   // EDGE chunk ranges of the unblocked order (aliased when nblk == 1)
        if (st != FALCON_OK) return st;
    }
    const uint64_t n = (uint64_t)g->n, m = (uint64_t)g->m;
    if (g->blk_bytes == 0) return FALCON_OK;
    uint64_t K = (4 * n + g->blk_bytes - 1) / g->blk_bytes;
    // at most 4 blocks: every block pass re-reads the frontier's row offsets
    // (rand-125M SSSP VERTEX: 8 blocks of 64 MB 54.6 ms, 4 of 128 MB 38.5 ms)
    if (K > MAX_BLOCKS_USED) K = MAX_BLOCKS_USED;
    while (K > 1 && K * (n + 1) >= (1ull << 32)) K--;
    if (K <= 1) return FALCON_OK;
    const uint32_t bsz = (uint32_t)(((n + K - 1) / K + 31) / 32 * 32);
    K = (n + bsz - 1) / bsz;
    if (K <= 1) return FALCON_OK;
    cudaStream_t s = g->stream;
    const uint64_t len = K * (n + 1);
    const uint32_t ntiles = (uint32_t)((len + 1023) / 1024);
    uint32_t *tiles = g->tiles;
    // built into locals, published only once complete (see ensure_src)
    uint32_t *rowb = nullptr, *srcb = nullptr, *perm_in = nullptr, *perm = nullptr;
    uint2 *cwb = nullptr, *chunkb = nullptr;
    uint8_t *keys = nullptr, *keys_out = nullptr;
    void *tmp = nullptr;
    auto undo = [&] {
        cudaStreamSynchronize(s);
        dfree(rowb); dfree(srcb); dfree(cwb); dfree(chunkb);
        dfree(keys); dfree(keys_out); dfree(perm_in); dfree(perm); dfree(tmp);
    };
#define BLK_TRY(call)                                                                             \
    do {                                                                                          \
        cudaError_t _e = (call);                                                                  \
        if (_e != cudaSuccess) {                                                                  \
            undo();                                                                               \
            return fail(_e == cudaErrorMemoryAllocation ? FALCON_ERR_NO_MEMORY : FALCON_ERR_CUDA, \
                        "destination-blocked layout: %s", cudaGetErrorString(_e));                \
        }                                                                                         \
    } while (0)
    BLK_TRY(dmalloc(&rowb, len));
    BLK_TRY(dmalloc(&cwb, m));
    BLK_TRY(dmalloc(&srcb, m));
    BLK_TRY(dmalloc(&chunkb, (size_t)((m + ECH_SSSP - 1) / ECH_SSSP)));
    k_blk_count<<<g->num_sms * 8, BLOCK, 0, s>>>((uint32_t)n, g->row_off, g->col, bsz, (uint32_t)K, rowb);
    k_scan_local<<<ntiles, 256, 0, s>>>(rowb, len, tiles);
    k_scan_tiles<<<1, 256, 0, s>>>(tiles, ntiles);
    k_scan_add<<<(unsigned)((len + 255) / 256), 256, 0, s>>>(rowb, len, tiles);
    {   // arcs grouped by target block, CSR order kept inside each block: a
        // stable radix sort of the arc indices by block id, then a gather
        size_t tmp_bytes = 0;
        int end_bit = 1;
        while ((1ull << end_bit) < K) end_bit++;
        BLK_TRY(dmalloc(&keys, m));
        BLK_TRY(dmalloc(&keys_out, m));
        BLK_TRY(dmalloc(&perm_in, m));
        BLK_TRY(dmalloc(&perm, m));
        k_blk_keys<<<g->num_sms * 8, BLOCK, 0, s>>>(m, g->col, bsz, keys, perm_in);
        BLK_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys_out, perm_in, perm, (int64_t)m, 0,
                                                end_bit, s));
        BLK_TRY(dev_alloc(&tmp, tmp_bytes));
        BLK_TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys_out, perm_in, perm, (int64_t)m, 0, end_bit,
                                                s));
        k_blk_gather<<<g->num_sms * 8, BLOCK, 0, s>>>(m, perm, g->cw, g->src, cwb, srcb);
        BLK_TRY(cudaStreamSynchronize(s));
        dfree(keys); dfree(keys_out); dfree(perm_in); dfree(perm); dfree(tmp);
        keys = keys_out = nullptr; perm_in = perm = nullptr; tmp = nullptr;
    }
    k_chunk_range<<<g->num_sms * 8, BLOCK, 0, s>>>((uint32_t)m, ECH_SSSP, srcb, chunkb);
    BLK_TRY(cudaGetLastError());
    BLK_TRY(cudaStreamSynchronize(s));
#undef BLK_TRY
    g->rowb = rowb; g->cwb = cwb; g->srcb = srcb; g->chunkb = chunkb;
    g->nblk = (uint32_t)K;
    g->bsz = bsz;
    return FALCON_OK;
}

// Reverse CSR (in-arcs: BFS pull, CC worklist), built once on the device: a
// stable LSD radix sort of the (target, source) arc pairs by target (CUB) --
// the in-row of v lists its sources in ascending order -- and the offsets
// read off the sorted targets.
falcon_status_t ensure_reverse(falcon_graph *g) {
    if (g->rin_off) return FALCON_OK;
    const uint64_t n = (uint64_t)g->n, m = (uint64_t)g->m;
    cudaStream_t s = g->stream;
    if (m) {
        falcon_status_t st = ensure_src(g);
        if (st != FALCON_OK) return st;
    }
    // built into locals, published only once complete (see ensure_src)
    uint32_t *rin_off = nullptr, *rin_col = nullptr, *keys_out = nullptr;
    void *tmp = nullptr;
    auto undo = [&] {
        cudaStreamSynchronize(s);
        dfree(rin_off); dfree(rin_col); dfree(keys_out); dfree(tmp);
    };
#define REV_TRY(call)                                                                             \
    do {                                                                                          \
        cudaError_t _e = (call);                                                                  \
        if (_e != cudaSuccess) {                                                                  \
            undo();                                                                               \
            return fail(_e == cudaErrorMemoryAllocation ? FALCON_ERR_NO_MEMORY : FALCON_ERR_CUDA, \
                        "reverse CSR: %s", cudaGetErrorString(_e));                               \
        }                                                                                         \
    } while (0)
    REV_TRY(dmalloc(&rin_off, n + 1));
    REV_TRY(dmalloc(&rin_col, m ? m : 1));
    if (!m) REV_TRY(cudaMemsetAsync(rin_off, 0, (n + 1) * 4, s));
    if (m) {
        int end_bit = 1;
        while (end_bit < 32 && (1ull << end_bit) < n) end_bit++;
        size_t tmp_bytes = 0;
        REV_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, g->col, keys_out, g->src, rin_col, (int64_t)m, 0,
                                                end_bit, s));
        REV_TRY(dmalloc(&keys_out, m));
        REV_TRY(dev_alloc(&tmp, tmp_bytes));
        REV_TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, g->col, keys_out, g->src, rin_col, (int64_t)m, 0,
                                                end_bit, s));
        // in-row offsets from the sorted targets (first position of every
        // target, vertices without in-arcs included) -- no atomics
        k_rin_off<<<g->num_sms * 8, BLOCK, 0, s>>>(m, (uint32_t)n, keys_out, rin_off);
        REV_TRY(cudaStreamSynchronize(s));
        dfree(keys_out);
        dfree(tmp);
        keys_out = nullptr; tmp = nullptr;
    }
    REV_TRY(cudaGetLastError());
    REV_TRY(cudaStreamSynchronize(s));
#undef REV_TRY
    g->rin_off = rin_off; g->rin_col = rin_col;
    return FALCON_OK;
}

falcon_status_t run_partitioned(falcon_graph *g, int algo, uint32_t source, int32_t *out, falcon_stats_t *stats);

// Drop the cached CUDA graphs (they bake in the launch arguments).
void drop_graphs(falcon_graph *g) {
    if (g->stream) cudaStreamSynchronize(g->stream);
    for (auto &row : g->execs)
        for (auto &x : row)
            if (x) { cudaGraphExecDestroy(x); x = nullptr; }
    for (auto &row : g->graphs)
        for (auto &x : row)
            if (x) { cudaGraphDestroy(x); x = nullptr; }
}

falcon_status_t run_launch(falcon_graph *g, int algo, uint32_t source, int style, int32_t *out);
falcon_status_t run_finish(falcon_graph *g, falcon_stats_t *stats);

// One call: launch (everything up to the asynchronous copies of the result
// and the control block) and finish (synchronise, statistics, status).
falcon_status_t run(falcon_graph *g, int algo, uint32_t source, int style, int32_t *out, falcon_stats_t *stats) {
    if (g && g->comm) {
        if (style < 0 || style > 3) return fail(FALCON_ERR_INVALID_ARG, "unknown style %d", style);
        if (style == DELTA && algo != SSSP) return fail(FALCON_ERR_INVALID_ARG, "FALCON_STYLE_DELTA is an SSSP schedule");
        return run_partitioned(g, algo, source, out, stats);
    }
    falcon_status_t st = run_launch(g, algo, source, style, out);
    if (st != FALCON_OK) return st;
    return run_finish(g, stats);
}

falcon_status_t run_launch(falcon_graph *g, int algo, uint32_t source, int style, int32_t *out) {
    if (g && g->comm) return fail(FALCON_ERR_UNSUPPORTED, "partitioned graphs run through falcon_sssp/bfs/cc");
    if (g && g->pend_algo >= 0) return fail(FALCON_ERR_INVALID_ARG, "a call is already in flight on this graph");
    if (!g) return fail(FALCON_ERR_INVALID_ARG, "graph is NULL");
    if (!out) return fail(FALCON_ERR_INVALID_ARG, "output pointer is NULL");
    if (style < 0 || style > 3) return fail(FALCON_ERR_INVALID_ARG, "unknown style %d", style);
    if (style == DELTA && algo != SSSP) return fail(FALCON_ERR_INVALID_ARG, "FALCON_STYLE_DELTA is an SSSP schedule");
    if (algo != CC && (int64_t)source >= g->n) return fail(FALCON_ERR_INVALID_ARG, "source %u >= n", source);
    CU(cudaSetDevice(g->device));
    // BFS WORKLIST on a sparse high-diameter graph runs as unit-weight
    // Δ-stepping with local continuation (R19): the hop
    // distance is the least fixpoint of MIN-relaxation with w = 1, whatever
    // the order.  The kernels are SSSP's over a (col, 1) copy of the arcs
    // (built on first use, 8 bytes per arc); the CUDA graph is cached in the
    // (BFS, DELTA) slot.  A view uses its parent's copy when there is one.
    falcon_graph *root = g->parent ? g->parent : g;
    // cw_unit is read here by the root and its views, possibly from several
    // host threads at once, and built by the root's first such call
    std::unique_lock<std::mutex> unit_lock(root->unit_mu);
    const bool unit = algo == BFS && style == WORKLIST &&
                      (g->bfs_unit > 0 || (g->bfs_unit < 0 && g->local_tiles && g->m < 3 * g->n)) &&
                      (!g->parent || root->cw_unit);
    g->unit_run = unit;
    if (!unit) unit_lock.unlock();
    if (unit) {
        style = DELTA;
        if (!root->cw_unit) {   // (only the root builds it; published once complete)
            uint2 *cu = nullptr;
            CU(dmalloc(&cu, (size_t)(g->m ? g->m : 1)));
            if (g->m) {
                int32_t *ones = nullptr;
                CU(dmalloc(&ones, (size_t)g->m));
                k_fill_i32<<<g->num_sms * 8, BLOCK, 0, g->stream>>>(ones, (uint64_t)g->m, 1);
                k_interleave<<<g->num_sms * 8, BLOCK, 0, g->stream>>>((uint64_t)g->m, g->col, ones, cu);
                CU(cudaStreamSynchronize(g->stream));
                dfree(ones);
            }
            root->cw_unit = cu;
        }
        g->cw_unit = root->cw_unit;
        unit_lock.unlock();
    }
    if (!g->parent) {   // a view shares layouts its parent built in graph_share
        if (style == EDGE) {
            falcon_status_t st = ensure_src(g);
            if (st != FALCON_OK) return st;
        }
        if (algo == SSSP && !unit) {
            falcon_status_t st = ensure_blocked(g);
            if (st != FALCON_OK) return st;
        }
        if ((algo == BFS && (style == VERTEX || (style == WORKLIST && g->wl_pull && !unit)) && g->pull_div) ||
            (algo == CC && style == WORKLIST)) {
            falcon_status_t st = ensure_reverse(g);
            if (st != FALCON_OK) return st;
        }
    }
    cudaStream_t s = g->stream;
    Args a = g->args();
    // round cap (R11): n + 2 (Bellman-Ford).  DELTA: SPEC.md:448's 10 n -- its
    // refill rounds are not bounded by one per bucket (a vertex parked in the
    // far set and later improved into the current bucket keeps its far bit and
    // comes back in a later refill), so 2 n + 4 was not a bound
    // (tests/test_overflow_gpu.py::test_delta_round_cap_chain).
    const int64_t capn = style == DELTA ? 10 * g->n + 16 : g->n + 2;
    const uint32_t cap = (uint32_t)(capn > 0xFFFFFFF0ll ? 0xFFFFFFF0ll : capn);
    uint32_t delta = 1;
    if (style == DELTA && !unit) {
        if (g->delta > 0) {
            delta = (uint32_t)g->delta;
        } else {
            if (!g->delta_auto) {   // average weight, once per graph
                unsigned long long *d_sum = nullptr, h_sum = 0;
                CU(dmalloc(&d_sum, 1));
                CU(cudaMemsetAsync(d_sum, 0, sizeof(unsigned long long), s));
                if (g->m) k_sum_weights<<<g->num_sms * 8, BLOCK, 0, s>>>((uint64_t)g->m, g->w, d_sum);
                CU(cudaMemcpyAsync(&h_sum, d_sum, sizeof h_sum, cudaMemcpyDeviceToHost, s));
                CU(cudaStreamSynchronize(s));
                dfree(d_sum);
                const unsigned long long avg = g->m ? h_sum / (unsigned long long)g->m : 1;
                g->delta_auto = (int32_t)(avg < 1 ? 1 : (avg > 0x3fffffff ? 0x3fffffff : avg));
            }
            delta = (uint32_t)g->delta_auto;
        }
    }
    CU(cudaEventRecord(g->ev0, s));
    if (algo == SSSP || unit) k_init<SSSP><<<g->grid_small, BLOCK, 0, s>>>(a, source, cap, 3u * g->cnt_slots, style, delta);
    else if (algo == BFS) k_init<BFS><<<g->grid_small, BLOCK, 0, s>>>(a, source, cap, 3u * g->cnt_slots, style, delta);
    else k_init<CC><<<g->grid_small, BLOCK, 0, s>>>(a, source, cap, 3u * g->cnt_slots, style, delta);
    CU(cudaGetLastError());

    double relax_ms = -1.0;
    int64_t relax_launches = 0;
    int64_t cc_passes = 0, cc_launches = 0;
    if (algo == CC) {
        // Fixed pass sequence (no fixpoint loop): union-find hooking is exact
        // after one pass over the arcs (cc.cuh).
        Tracer tr{g};
        Tracer *t = g->profiling ? &tr : nullptr;
        auto relax_mark = [&](const char *nm) { if (t) t->mark(s, nm, 0); };
        auto other_mark = [&](const char *nm) { if (t) t->mark(s, nm, 1); };
        other_mark("begin");
        if (style == VERTEX) {
            launch_l2(g, k_cc_vertex<BLOCK>, g->grid_cc, s, a);
            relax_mark("cc_vertex");
            cc_passes = 1;
        } else if (style == EDGE) {
            launch_l2(g, k_cc_edge<BLOCK>, g->grid_small, s, a);
            relax_mark("cc_edge");
            cc_passes = 1;
        } else {
            launch_l2(g, k_cc_vertex<BLOCK, 2>, g->grid_cc, s, a);   // sampling: first 2 arcs of every row
            relax_mark("cc_sample");
            launch_l2(g, k_compress, g->grid_small, s, a);
            other_mark("compress");
            k_cc_giant<<<1, 1024, 0, s>>>(a);
            other_mark("cc_giant");
            launch_l2(g, k_cc_rest<BLOCK>, g->grid_cc, s, a);
            relax_mark("cc_rest");
            cc_passes = 2;
            cc_launches += 4;
        }
        launch_l2(g, k_compress, g->grid_small, s, a);
        other_mark("compress");
        cc_launches += 2;
        CU(cudaGetLastError());
        if (t) {
            relax_ms = 0.0;
            for (size_t i = 1; i < tr.marks.size(); i++) {
                float ms = 0.f;
                CU(cudaEventSynchronize(tr.marks[i].ev));
                CU(cudaEventElapsedTime(&ms, tr.marks[i - 1].ev, tr.marks[i].ev));
                if (tr.marks[i].kind == 0) { relax_ms += ms; relax_launches++; }
            }
        }
    } else if (!g->profiling) {
        falcon_status_t st = build_graph(g, algo, style);
        if (st != FALCON_OK) return st;
        CU(cudaGraphLaunch(g->execs[algo][style], s));
    } else {
        // Host-driven loop with a CUDA event after every launch (same kernels).
        const char *trace_env = getenv("FALCON_TRACE");
        const bool trace = trace_env && trace_env[0] == '1';
        Tracer tr{g};
        std::vector<uint32_t> fr_len;   // trace: frontier length after each round
        for (;;) {
            const int per_check = trace ? 1 : HOST_CHECK_EVERY;
            for (int k = 0; k < per_check; k++) {
                tr.round++;
                launch_round(g, algo, style, s, 0, 0, &tr);
            }
            CU(cudaGetLastError());
            CU(cudaMemcpyAsync(g->h_ctrl, g->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s));
            CU(cudaStreamSynchronize(s));
            if (trace) fr_len.push_back(g->h_ctrl->in_len);
            if (g->h_ctrl->done) break;
        }
        const uint32_t rounds = g->h_ctrl->iter;
        relax_ms = 0.0;
        std::vector<std::string> lines;
        for (size_t i = 1; i < tr.marks.size(); i++) {
            const auto &m = tr.marks[i];
            if (m.round > rounds || std::strcmp(m.name, "begin") == 0) continue;
            float t = 0.f;
            CU(cudaEventElapsedTime(&t, tr.marks[i - 1].ev, m.ev));
            if (m.kind == 0) relax_ms += t;
            if (std::strcmp(m.name, "expand") == 0 || std::strcmp(m.name, "edge") == 0) relax_launches++;
            if (trace) {
                char buf[160];
                snprintf(buf, sizeof buf, "round %4u %-9s %9.1f us%s", m.round, m.name, 1e3 * t,
                         std::strcmp(m.name, "advance") == 0 && m.round - 1 < fr_len.size()
                             ? (" | frontier after round: " + std::to_string(fr_len[m.round - 1])).c_str() : "");
                lines.push_back(buf);
            }
        }
        if (trace)
            for (auto &l : lines) fprintf(stderr, "[falcon trace] %s\n", l.c_str());
    }
    if (algo == BFS && !unit) k_bfs_levels<<<g->grid_small, BLOCK, 0, s>>>(a);   // byte levels -> val
    k_finish<<<1, BLOCK, 0, s>>>(a, (uint32_t)g->cnt_slots);
    CU(cudaGetLastError());
    CU(cudaEventRecord(g->ev1, s));
    // A copy into pageable host memory would block this thread until the call
    // completes (falcon_run_many launches every job before waiting on any):
    // it is deferred to run_finish.  Device and pinned outputs copy here.
    cudaPointerAttributes pa{};
    const bool pageable = cudaPointerGetAttributes(&pa, out) != cudaSuccess || pa.type == cudaMemoryTypeUnregistered;
    cudaGetLastError();   // (an unregistered pointer may leave an error on older runtimes)
    g->pend_out = pageable ? out : nullptr;
    if (!pageable) CU(cudaMemcpyAsync(out, g->val, (size_t)g->n * sizeof(int32_t), cudaMemcpyDefault, s));
    CU(cudaMemcpyAsync(g->h_ctrl, g->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s));
    g->pend_algo = algo;
    g->pend_cap = cap;
    g->pend_relax_ms = relax_ms;
    g->pend_relax_launches = relax_launches;
    g->pend_cc_passes = cc_passes;
    g->pend_cc_launches = cc_launches;
    return FALCON_OK;
}

// Overflow (reading R3): candidates >= INF are dropped during the fixpoint;
// afterwards this decides, independent of the schedule, whether a reachable
// vertex was left at INF (k_overflow_check), exactly when the oracle reports
// a finite shortest distance >= INF.  Runs only after such a candidate.
falcon_status_t overflow_certificate(falcon_graph *g, const uint32_t *row_off, const uint32_t *col, const int32_t *val,
                                     bool *bad) {
    cudaStream_t s = g->stream;
    int flag = 0;
    CU(cudaMemsetAsync(g->d_flags, 0, sizeof(int), s));
    k_overflow_check<<<g->num_sms * 8, BLOCK, 0, s>>>((uint32_t)g->n, row_off, col, val, g->d_flags);
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(&flag, g->d_flags, sizeof(int), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    *bad = flag != 0;
    return FALCON_OK;
}

falcon_status_t run_finish(falcon_graph *g, falcon_stats_t *stats) {
    if (g->pend_algo < 0) return fail(FALCON_ERR_INVALID_ARG, "no call in flight on this graph");
    const int algo = g->pend_algo;
    g->pend_algo = -1;
    CU(cudaSetDevice(g->device));
    CU(cudaStreamSynchronize(g->stream));
    if (g->pend_out) {   // pageable host output (run_launch)
        int32_t *o = g->pend_out;
        g->pend_out = nullptr;
        CU(cudaMemcpy(o, g->val, (size_t)g->n * sizeof(int32_t), cudaMemcpyDeviceToHost));
    }
    const Ctrl &c = *g->h_ctrl;
    if (stats) {
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, g->ev0, g->ev1));
        stats->iterations = algo == CC ? g->pend_cc_passes : c.iter;
        stats->vertices_processed = (int64_t)c.vertices;
        stats->edges_relaxed = (int64_t)c.edges;
        stats->updates = (int64_t)c.updates;
        stats->kernel_launches = (int64_t)c.launches + g->pend_cc_launches;
        stats->ms = ms;
        stats->relax_ms = g->pend_relax_ms;
        stats->relax_launches = g->pend_relax_launches;
    }
    if (c.status == ST_NOT_CONVERGED)
        return fail(FALCON_ERR_NOT_CONVERGED, "no fixpoint within %u rounds", g->pend_cap);
    if (c.status == ST_QUEUE) return fail(FALCON_ERR_CUDA, "internal error: frontier queue bound exceeded");
    if (algo == SSSP && c.cand_ovf) {   // some candidate reached INF: is a reachable vertex left at INF? (R3)
        bool bad = false;
        falcon_status_t st = overflow_certificate(g, g->row_off, g->col, g->val, &bad);
        if (st != FALCON_OK) return st;
        if (bad) return fail(FALCON_ERR_OVERFLOW, "a finite shortest distance is >= FALCON_INF");
    }
    g_last_error.clear();
    return FALCON_OK;
}

// Minimum spanning forest (mst.cuh): Borůvka rounds, each checked on the
// host (at most log2(n) + 1 rounds).
falcon_status_t run_mst(falcon_graph *g, int style, int64_t *total, int64_t *nedges, int32_t *label_out,
                        falcon_stats_t *stats) {
    if (!g || !total) return fail(FALCON_ERR_INVALID_ARG, "graph or total is NULL");
    if (g->comm) return fail(FALCON_ERR_UNSUPPORTED, "falcon_mst on a partitioned graph");
    if (style != VERTEX && style != EDGE)
        return fail(FALCON_ERR_UNSUPPORTED, "falcon_mst runs VERTEX or EDGE style (Borůvka is arc-parallel)");
    if (g->pend_algo >= 0) return fail(FALCON_ERR_INVALID_ARG, "a call is already in flight on this graph");
    CU(cudaSetDevice(g->device));
    g->unit_run = false;
    if (!g->parent) {
        falcon_status_t st = ensure_src(g);
        if (st != FALCON_OK) return st;
    }
    if (!g->mst_best) CU(dmalloc(&g->mst_best, (size_t)g->n));
    // live lists (EDGE: arc indices, VERTEX: vertices), ping-pong
    const size_t lcap = (size_t)(style == EDGE ? g->m : g->n) + 1;
    if (g->mst_lcap < lcap) {
        dfree(g->mst_list);
        g->mst_list = nullptr;
        CU(dmalloc(&g->mst_list, 2 * lcap));
        g->mst_lcap = lcap;
    }
    cudaStream_t s = g->stream;
    Args a = g->args();
    const int gs = g->grid_small;
    CU(cudaEventRecord(g->ev0, s));
    k_init<CC><<<gs, BLOCK, 0, s>>>(a, 0, 64, 3u * g->cnt_slots, VERTEX, 1);   // comp[v] = v
    int64_t rounds = 0, launches = 2, hooks = 0;
    const uint32_t *in = nullptr;   // first round: every vertex / arc
    uint32_t nin = 0;
    bool collect = false;           // write this round's live list (else only count it)
    for (;;) {
        uint32_t *out = collect ? g->mst_list + (rounds & 1) * g->mst_lcap : nullptr;
        k_mst_reset<<<gs, BLOCK, 0, s>>>(a, g->mst_best);
        if (style == VERTEX) k_mst_min_vertex<BLOCK><<<g->grid_cc, BLOCK, 0, s>>>(a, g->mst_best, in, nin, out);
        else k_mst_min_edge<BLOCK><<<gs, BLOCK, 0, s>>>(a, g->mst_best, in, nin, out);
        k_mst_hook<BLOCK><<<gs, BLOCK, 0, s>>>(a, g->mst_best, g->fr0);
        k_mst_apply<<<gs, BLOCK, 0, s>>>(a, g->fr0);
        launch_l2(g, k_compress, gs, s, a);
        launches += 5;
        rounds++;
        CU(cudaGetLastError());
        CU(cudaMemcpyAsync(g->h_ctrl, g->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        hooks += g->h_ctrl->hooks;
        if (g->h_ctrl->hooks == 0) break;
        if (rounds > 64) return fail(FALCON_ERR_NOT_CONVERGED, "Borůvka did not converge in 64 rounds");
        // the live list replaces a full scan once it is short (indirect
        // gathers cost more than streaming while most arcs are still live)
        nin = g->h_ctrl->found;   // live items of this round (the list holds them if collected)
        in = out && (uint64_t)nin * 4 < lcap ? out : nullptr;
        collect = (uint64_t)nin * 2 < lcap;
    }
    uint32_t *minid = reinterpret_cast<uint32_t *>(g->mst_best);
    CU(cudaMemsetAsync(minid, 0xff, (size_t)g->n * 4, s));
    k_mst_minid<<<gs, BLOCK, 0, s>>>(a, minid);
    k_mst_label<<<gs, BLOCK, 0, s>>>(a, minid);
    k_finish<<<1, BLOCK, 0, s>>>(a, (uint32_t)g->cnt_slots);
    launches += 3;
    CU(cudaGetLastError());
    CU(cudaEventRecord(g->ev1, s));
    if (label_out) CU(cudaMemcpyAsync(label_out, g->val, (size_t)g->n * sizeof(int32_t), cudaMemcpyDefault, s));
    CU(cudaMemcpyAsync(g->h_ctrl, g->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    const Ctrl &c = *g->h_ctrl;
    *total = (int64_t)c.wsum;
    if (nedges) *nedges = hooks;
    if (stats) {
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, g->ev0, g->ev1));
        stats->iterations = rounds;
        stats->vertices_processed = (int64_t)g->n * rounds;
        stats->edges_relaxed = (int64_t)c.edges;
        stats->updates = hooks;
        stats->kernel_launches = launches;
        stats->ms = ms;
        stats->relax_ms = -1.0;
        stats->relax_launches = 0;
    }
    g_last_error.clear();
    return FALCON_OK;
}

void destroy_partitioned(falcon_graph *g);

void destroy(falcon_graph *g) {
    if (!g) return;
    if (g->comm) {
        destroy_partitioned(g);
        delete g;
        return;
    }
    cudaSetDevice(g->device);
    if (g->stream) cudaStreamSynchronize(g->stream);
    if (g->parent) {   // a view: the arrays below belong to the parent
        g->parent->nviews--;
        g->row_off = g->col = g->src = g->rowb = g->srcb = g->rin_off = g->rin_col = g->tiles = nullptr;
        g->w = nullptr; g->cw = g->cwb = g->chunk = g->chunkb = g->chunks = g->cw_unit = nullptr;
    }
    for (auto &row : g->execs)
        for (auto &x : row)
            if (x) cudaGraphExecDestroy(x);
    for (auto &row : g->graphs)
        for (auto &x : row)
            if (x) cudaGraphDestroy(x);
    for (auto e : g->pev) cudaEventDestroy(e);
    if (g->ev0) cudaEventDestroy(g->ev0);
    if (g->ev1) cudaEventDestroy(g->ev1);
    for (void *p : {(void *)g->row_off, (void *)g->col, (void *)g->w, (void *)g->cw, (void *)g->src,
                    (void *)g->rin_off, (void *)g->rin_col, (void *)g->rowb, (void *)g->cwb, (void *)g->srcb,
                    (void *)g->chunk, (void *)g->chunkb, (void *)g->chunks, (void *)g->val, (void *)g->lv8, (void *)g->bm,
                    (void *)g->fr0, (void *)g->fr1, (void *)g->tiles, (void *)g->ctrl, (void *)g->cnt,
                    (void *)g->d_flags, (void *)g->mst_best, (void *)g->mst_list, (void *)g->xcounts,
                    (void *)g->xcnt_recv, (void *)g->outbox, (void *)g->inbox, (void *)g->bounds_d,
                    (void *)g->d_outboxes, (void *)g->d_counts, (void *)g->cw_unit})
        dfree(p);   // back to the device cache (the stream was synchronised above)
    host_ctrl_free(g->h_ctrl);
    if (g->cap_stream) cudaStreamDestroy(g->cap_stream);
    if (g->own_stream && g->stream) cudaStreamDestroy(g->stream);
    delete g;
}

falcon_status_t load(int64_t n, int64_t m, const uint32_t *row_off, const uint32_t *col, const int32_t *w,
                     const falcon_load_opts_t *opts, falcon_graph *g) {
    int dev = opts ? opts->device : -1;
    if (dev < 0) CU(cudaGetDevice(&dev));
    g->device = dev;
    CU(cudaSetDevice(dev));
    CU(cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, dev));
    if (opts && opts->cuda_stream) {
        g->stream = (cudaStream_t)opts->cuda_stream;
    } else {
        CU(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
        g->own_stream = true;
    }
    CU(cudaStreamCreateWithFlags(&g->cap_stream, cudaStreamNonBlocking));
    CU(cudaEventCreate(&g->ev0));
    CU(cudaEventCreate(&g->ev1));
    g->n = n; g->m = m;
    cudaStream_t s = g->stream;

    CU(dmalloc(&g->row_off, (size_t)n + 1));
    CU(dmalloc(&g->col, (size_t)m));
    CU(dmalloc(&g->w, (size_t)m));
    CU(dmalloc(&g->val, (size_t)n));
    CU(dmalloc(&g->lv8, ((size_t)n + 15) / 16 * 16 + 16));
    g->nwords = (uint32_t)((((n + 31) / 32) + 3) & ~3ll);
    CU(dmalloc(&g->bm, 4 * (size_t)g->nwords));
    CU(dmalloc(&g->fr0, (size_t)n + 1));
    CU(dmalloc(&g->fr1, (size_t)n + 1));   // n+1: doubles as the reverse-CSR cursor at build time
    CU(dmalloc(&g->tiles, (size_t)(MAX_BLK * ((uint64_t)n + 1) + 1023) / 1024 + 1));   // scan tile sums
    CU(dmalloc(&g->ctrl, 1));
    CU(cudaMemsetAsync(g->ctrl, 0, sizeof(Ctrl), s));   // padding / unused fields: the whole block is copied out
    CU(dmalloc(&g->d_flags, 1));
    CU(host_ctrl_alloc(reinterpret_cast<void **>(&g->h_ctrl), sizeof(Ctrl)));

    CU(cudaMemcpyAsync(g->row_off, row_off, ((size_t)n + 1) * 4, cudaMemcpyDefault, s));
    if (m) CU(cudaMemcpyAsync(g->col, col, (size_t)m * 4, cudaMemcpyDefault, s));
    if (m && w) CU(cudaMemcpyAsync(g->w, w, (size_t)m * 4, cudaMemcpyDefault, s));
    if (m && !w) k_fill_i32<<<g->num_sms * 8, BLOCK, 0, s>>>(g->w, (uint64_t)m, 1);
    CU(dmalloc(&g->cw, (size_t)m));
    if (m) k_interleave<<<g->num_sms * 8, BLOCK, 0, s>>>((uint64_t)m, g->col, g->w, g->cw);

    // grid sizes: a multiple of the SM count x resident CTAs, capped by the work
    int occ_f = 0, occ_e = 0, occ_p = 0;
    const char *var = getenv("FALCON_EXPAND_VARIANT");
    g->variant = var ? atoi(var) : 0;
    static const int var_minb[7] = {3, 4, 3, 6, 2, 4, 4};
    occ_f = var_minb[g->variant >= 0 && g->variant < 7 ? g->variant : 0];
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_p, k_persist<SSSP, DELTA, BLOCK, UNROLL>, BLOCK, 0));
    {
        int o2 = 0;
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_persist<BFS, WORKLIST, BLOCK, UNROLL>, BLOCK, 0));
        if (o2 < occ_p) occ_p = o2;
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_persist<SSSP, WORKLIST, BLOCK, UNROLL>, BLOCK, 0));
        if (o2 < occ_p) occ_p = o2;
    }
    const char *pe = getenv("FALCON_PERSIST");
    g->persist = (pe && pe[0] == '1') && occ_p > 0;   // measured: no faster than per-round graph launches
    const char *pm = getenv("FALCON_PERSIST_MAX");
    if (pm) g->persist_max = (uint32_t)atoll(pm);
    int occ_eb = 0;
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_e, k_edge<SSSP, BLOCK, EDGE_QP_SSSP>, BLOCK, 0));
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_eb, k_edge<BFS, BLOCK, EDGE_QP_BFS>, BLOCK, 0));
    auto clampg = [](int64_t want, int64_t cap) { return (int)(want < 1 ? 1 : (want > cap ? cap : want)); };
    auto full = [&](int occ) { return (int64_t)g->num_sms * (occ > 0 ? occ : 1); };
    g->grid_persist = (int)full(occ_p);
    g->grid_expand_fr = clampg((n + BLOCK - 1) / BLOCK, full(occ_f));
    g->grid_expand_dl = clampg((n + BLOCK - 1) / BLOCK, full(g->variant ? occ_f : 4));
    g->grid_edge = clampg((m / 4 + 1 + BLOCK * EDGE_QP_SSSP - 1) / (BLOCK * EDGE_QP_SSSP), full(occ_e));
    g->grid_edge_b = clampg((m / 4 + 1 + BLOCK * EDGE_QP_BFS - 1) / (BLOCK * EDGE_QP_BFS), full(occ_eb));
    g->grid_small = clampg((n + BLOCK - 1) / BLOCK, (int64_t)g->num_sms * 8);
    g->grid_cc = clampg((n + BLOCK - 1) / BLOCK, (int64_t)g->num_sms * 8);
    g->grid_pull = clampg(((int64_t)g->nwords * 32 + BLOCK - 1) / BLOCK, (int64_t)g->num_sms * 8);
    if (const char *bmb = getenv("FALCON_BLOCK_MB")) g->blk_bytes = (size_t)atoll(bmb) << 20;   // 0: no blocking
    if (const char *dd = getenv("FALCON_DENSE_DIV")) g->dense_div = (uint32_t)atoi(dd);        // 0: never dense
    if (const char *wq = getenv("FALCON_WL_NOQ")) g->wl_noq = (uint32_t)atoi(wq);
    if (const char *dq = getenv("FALCON_DL_NOQ")) g->dl_noq = (uint32_t)atoi(dq);
    if (const char *sd = getenv("FALCON_SPLIT_DIV")) g->split_div = (uint32_t)atoi(sd);
    if (m < 3 * n) { g->local_tiles = 16; g->local_max = 0xffffffffu; g->wl_local_tiles = 4; }
    else if (m >= 6 * n) g->local_tiles = 0;   // dense / skewed (rmat): measured no gain
    if (const char *lt = getenv("FALCON_WL_LOCAL")) g->wl_local_tiles = (uint32_t)atoi(lt);
    if (const char *dc = getenv("FALCON_DELTA_CAP")) g->delta_cap = (uint32_t)atoi(dc);
    if (const char *lm = getenv("FALCON_WL_LOCAL_MAX")) g->wl_local_max = (uint32_t)atoll(lm);
    if (const char *lt = getenv("FALCON_LOCAL")) g->local_tiles = (uint32_t)atoi(lt);
    if (const char *lm = getenv("FALCON_LOCAL_MAX")) g->local_max = (uint32_t)atoll(lm);
    if (const char *bu = getenv("FALCON_BFS_UNIT")) g->bfs_unit = (int32_t)atoi(bu);
    if (const char *bd = getenv("FALCON_BLOCK_DIV")) g->blk_div = (uint32_t)atoi(bd);          // 0: never blocked
    const char *pd = getenv("FALCON_BFS_PULL_DIV");
    if (pd) g->pull_div = (uint32_t)atoi(pd);
    if (const char *pu = getenv("FALCON_BFS_PULL_RULE")) g->pull_rule = (uint32_t)atoi(pu);
    if (const char *ct = getenv("FALCON_CTA_THR")) g->cta_thr = (uint32_t)atoi(ct);
    if (const char *sn = getenv("FALCON_SKIP_NOW")) g->skip_now = (uint32_t)atoi(sn);
    if (const char *wp = getenv("FALCON_BFS_WL_PULL")) g->wl_pull = (uint32_t)atoi(wp);
    if (const char *lv = getenv("FALCON_BFS_LAZY_DIV")) g->lazy_div = (uint32_t)atoi(lv);
    int slots = g->grid_persist;
    for (int gsz : {g->grid_expand_fr, g->grid_expand_dl, g->grid_edge, g->grid_edge_b, g->grid_small, g->grid_cc,
                    g->grid_pull})
        if (gsz > slots) slots = gsz;
    g->cnt_slots = slots;
    CU(dmalloc(&g->cnt, 3 * (size_t)slots));

    // Persisting L2 window over the gathered value array: opt-in
    // (FALCON_L2_PERSIST=1).  Measured on B200 it costs more than it gains
    // (rand-25M: SSSP VERTEX 4.74 -> 4.98 ms, BFS WORKLIST 1.70 -> 2.10 ms
    // with the window): the reserved lines crowd out the bitmaps and queues.
    const char *env = getenv("FALCON_L2_PERSIST");
    if (env && env[0] == '1') {
        int max_persist = 0, max_window = 0;
        cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
        cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev);
        if (max_persist > 0 && max_window > 0) {
            size_t cur = 0;
            cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
            if (cur < (size_t)max_persist) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)max_persist);
            const size_t bytes = (size_t)n * sizeof(int32_t);
            g->apw.base_ptr = g->val;
            g->apw.num_bytes = bytes < (size_t)max_window ? bytes : (size_t)max_window;
            const double ratio = (double)max_persist / (double)g->apw.num_bytes;
            g->apw.hitRatio = (float)(ratio < 1.0 ? ratio : 1.0);
            g->apw.hitProp = cudaAccessPropertyPersisting;
            g->apw.missProp = cudaAccessPropertyStreaming;
            g->l2_window = true;
        }
        cudaGetLastError();
    }

    CU(cudaMemsetAsync(g->d_flags, 0, sizeof(int), s));
    k_validate<<<g->num_sms * 8, BLOCK, 0, s>>>((uint32_t)n, (uint32_t)m, g->row_off, g->col, w ? g->w : nullptr,
                                                 g->d_flags);
    CU(cudaGetLastError());
    int flags = 0;
    CU(cudaMemcpyAsync(&flags, g->d_flags, sizeof(int), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    if (flags & 1) return fail(FALCON_ERR_OUT_OF_RANGE, "row_off must start at 0, be nondecreasing and end at m");
    if (flags & 2) return fail(FALCON_ERR_OUT_OF_RANGE, "col[e] >= n");
    if (flags & 4) return fail(FALCON_ERR_OUT_OF_RANGE, "negative weight");
    if (opts && (opts->flags & FALCON_LOAD_BUILD_REVERSE)) {
        falcon_status_t st = ensure_reverse(g);
        if (st != FALCON_OK) return st;
    }
    if (opts && (opts->flags & FALCON_LOAD_BUILD_COO)) {
        falcon_status_t st = ensure_src(g);
        if (st != FALCON_OK) return st;
        CU(cudaStreamSynchronize(s));
    }
    return FALCON_OK;
}

// graph_share: a view of `p` -- its read-only graph arrays (CSR, COO, chunk
// ranges, blocked layout, reverse CSR: all built here, once, on the parent)
// and its own scratch (value array, bitmaps, queues, control block, counters,
// stream, CUDA graphs), so calls on the parent and on its views may run at
// the same time (falcon_run_many; the paper's concurrent kernels,
// PAPER.md:1040-1064).
falcon_status_t share(falcon_graph *p, const falcon_load_opts_t *opts, falcon_graph *v) {
    CU(cudaSetDevice(p->device));
    falcon_status_t st = ensure_src(p);
    if (st == FALCON_OK) st = ensure_blocked(p);
    if (st == FALCON_OK) st = ensure_reverse(p);
    if (st != FALCON_OK) return st;
    v->parent = p;
    v->device = p->device;
    v->n = p->n; v->m = p->m;
    v->row_off = p->row_off; v->col = p->col; v->src = p->src; v->w = p->w; v->cw = p->cw;
    v->rowb = p->rowb; v->srcb = p->srcb; v->cwb = p->cwb;
    v->chunk = p->chunk; v->chunkb = p->chunkb; v->chunks = p->chunks;
    v->nblk = p->nblk; v->bsz = p->bsz; v->blk_bytes = p->blk_bytes;
    v->dense_div = p->dense_div; v->blk_div = p->blk_div; v->wl_noq = p->wl_noq; v->dl_noq = p->dl_noq; v->split_div = p->split_div; v->local_tiles = p->local_tiles; v->local_max = p->local_max;
    v->wl_local_tiles = p->wl_local_tiles; v->wl_local_max = p->wl_local_max; v->delta_cap = p->delta_cap;
    v->bfs_unit = p->bfs_unit;
    v->rin_off = p->rin_off; v->rin_col = p->rin_col; v->pull_div = p->pull_div; v->pull_rule = p->pull_rule; v->cta_thr = p->cta_thr; v->lazy_div = p->lazy_div;
    v->skip_now = p->skip_now; v->wl_pull = p->wl_pull;
    v->nwords = p->nwords; v->num_sms = p->num_sms;
    v->grid_persist = p->grid_persist; v->grid_expand_fr = p->grid_expand_fr; v->grid_expand_dl = p->grid_expand_dl;
    v->grid_pull = p->grid_pull; v->grid_cc = p->grid_cc; v->grid_edge = p->grid_edge; v->grid_edge_b = p->grid_edge_b;
    v->grid_small = p->grid_small; v->cnt_slots = p->cnt_slots;
    v->delta = p->delta; v->delta_auto = p->delta_auto; v->variant = p->variant;
    v->persist = p->persist; v->persist_max = p->persist_max;
    p->nviews++;
    if (opts && opts->cuda_stream) {
        v->stream = (cudaStream_t)opts->cuda_stream;
    } else {
        CU(cudaStreamCreateWithFlags(&v->stream, cudaStreamNonBlocking));
        v->own_stream = true;
    }
    CU(cudaStreamCreateWithFlags(&v->cap_stream, cudaStreamNonBlocking));
    CU(cudaEventCreate(&v->ev0));
    CU(cudaEventCreate(&v->ev1));
    const size_t n = (size_t)p->n;
    CU(dmalloc(&v->val, n));
    CU(dmalloc(&v->lv8, (n + 15) / 16 * 16 + 16));
    CU(dmalloc(&v->bm, 4 * (size_t)v->nwords));
    CU(dmalloc(&v->fr0, n + 1));
    CU(dmalloc(&v->fr1, n + 1));
    CU(dmalloc(&v->ctrl, 1));
    CU(cudaMemsetAsync(v->ctrl, 0, sizeof(Ctrl), v->stream));
    CU(dmalloc(&v->cnt, 3 * (size_t)v->cnt_slots));
    CU(dmalloc(&v->d_flags, 1));   // the view's own (overflow certificate)
    CU(host_ctrl_alloc(reinterpret_cast<void **>(&v->h_ctrl), sizeof(Ctrl)));
    v->l2_window = p->l2_window;
    v->apw = p->apw;
    v->apw.base_ptr = v->val;
    return FALCON_OK;
}

}  // namespace

#include "partition.cuh"

extern "C" {

falcon_status_t graph_load_csr(int64_t n, int64_t m, const uint32_t *row_off, const uint32_t *col, const int32_t *w,
                               const falcon_load_opts_t *opts, falcon_graph_t **out) {
    NvtxRange r("graph_load_csr");
    if (!out) return fail(FALCON_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    const bool slice = opts && (opts->flags & FALCON_LOAD_SLICE);   // a rank's slice may be empty
    if (n < (slice ? 0 : 1) || n >= (1ll << 31)) return fail(FALCON_ERR_INVALID_ARG, "n must be in [1, 2^31)");
    if (m < 0 || m >= (1ll << 32)) return fail(FALCON_ERR_INVALID_ARG, "m must be in [0, 2^32)");
    if (!row_off || (m > 0 && !col)) return fail(FALCON_ERR_INVALID_ARG, "row_off/col is NULL");
    if (opts && (opts->flags & ~(uint32_t)(FALCON_LOAD_BUILD_COO | FALCON_LOAD_BUILD_REVERSE | FALCON_LOAD_SLICE |
                                           FALCON_LOAD_GATHER)))
        return fail(FALCON_ERR_UNSUPPORTED, "unknown load flags 0x%x", opts->flags);
    if (opts && !opts->comm && (opts->flags & (FALCON_LOAD_SLICE | FALCON_LOAD_GATHER)))
        return fail(FALCON_ERR_INVALID_ARG, "FALCON_LOAD_SLICE / FALCON_LOAD_GATHER need a communicator");
    falcon_graph *g = new (std::nothrow) falcon_graph();
    if (!g) return fail(FALCON_ERR_NO_MEMORY, "host allocation failed");
    falcon_status_t st = (opts && opts->comm) ? load_partitioned(n, m, row_off, col, w, opts, g)
                                              : load(n, m, row_off, col, w, opts, g);
    if (st != FALCON_OK) {
        std::string msg = g_last_error;
        destroy(g);
        g_last_error = msg;
        return st;
    }
    g_last_error.clear();
    *out = g;
    return FALCON_OK;
}

falcon_status_t graph_free(falcon_graph_t *g) {
    if (g && g->nviews > 0) return fail(FALCON_ERR_INVALID_ARG, "graph has %d live views (free them first)", g->nviews.load());
    destroy(g);
    return FALCON_OK;
}

falcon_status_t falcon_trim_memory(int64_t *released_bytes) {
    DevCache &c = dev_cache();
    std::vector<void *> rel;
    int64_t bytes = 0;
    {
        std::lock_guard<std::mutex> lk(c.mu);
        for (auto &kv : c.idle) { rel.push_back(kv.second); bytes += (int64_t)kv.first.second; }
        c.idle.clear();
    }
    for (void *q : rel) cudaFree(q);
    if (released_bytes) *released_bytes = bytes;
    return FALCON_OK;
}

falcon_status_t graph_share(falcon_graph_t *g, const falcon_load_opts_t *opts, falcon_graph_t **out) {
    if (!g || !out) return fail(FALCON_ERR_INVALID_ARG, "graph or out is NULL");
    *out = nullptr;
    if (g->comm) return fail(FALCON_ERR_UNSUPPORTED, "graph_share of a partitioned graph");
    falcon_graph *root = g->parent ? g->parent : g;   // a view of a view shares the root's arrays
    falcon_graph *v = new (std::nothrow) falcon_graph();
    if (!v) return fail(FALCON_ERR_NO_MEMORY, "host allocation failed");
    falcon_status_t st = share(root, opts, v);
    if (st != FALCON_OK) {
        std::string msg = g_last_error;
        if (v->parent) destroy(v); else delete v;
        g_last_error = msg;
        return st;
    }
    g_last_error.clear();
    *out = v;
    return FALCON_OK;
}

falcon_status_t falcon_run_many(int njobs, falcon_graph_t *const *graphs, const falcon_job_t *jobs,
                                int32_t *const *outs, falcon_stats_t *stats) {
    NvtxRange r("falcon_run_many");
    if (njobs < 0 || (njobs > 0 && (!graphs || !jobs || !outs))) return fail(FALCON_ERR_INVALID_ARG, "bad job arrays");
    for (int i = 0; i < njobs; i++) {
        if (!graphs[i]) return fail(FALCON_ERR_INVALID_ARG, "job %d: graph is NULL", i);
        if (graphs[i]->comm) return fail(FALCON_ERR_UNSUPPORTED, "job %d: partitioned graph", i);
        if (jobs[i].algo < FALCON_ALGO_SSSP || jobs[i].algo > FALCON_ALGO_CC)
            return fail(FALCON_ERR_INVALID_ARG, "job %d: unknown algorithm %d", i, (int)jobs[i].algo);
        for (int j = 0; j < i; j++)
            if (graphs[j] == graphs[i])
                return fail(FALCON_ERR_INVALID_ARG, "jobs %d and %d share a graph handle (use graph_share)", j, i);
    }
    int launched = 0;
    falcon_status_t first = FALCON_OK;
    std::string msg;
    for (; launched < njobs; launched++) {   // every job is in flight before any is waited on
        const falcon_job_t &J = jobs[launched];
        falcon_status_t st = run_launch(graphs[launched], (int)J.algo, J.source, (int)J.style, outs[launched]);
        if (st != FALCON_OK) { first = st; msg = g_last_error; break; }
    }
    for (int i = 0; i < launched; i++) {
        falcon_status_t st = run_finish(graphs[i], stats ? stats + i : nullptr);
        if (st != FALCON_OK && first == FALCON_OK) { first = st; msg = g_last_error; }
    }
    if (first != FALCON_OK) { g_last_error = msg; return first; }
    g_last_error.clear();
    return FALCON_OK;
}

falcon_status_t graph_exchange_bytes(const falcon_graph_t *g, int64_t *bytes) {
    if (!g || !bytes) return fail(FALCON_ERR_INVALID_ARG, "graph or bytes is NULL");
    *bytes = g->comm ? (int64_t)g->xbytes : 0;
    return FALCON_OK;
}

falcon_status_t graph_partition_info(const falcon_graph_t *g, int32_t *exchange_mode, int64_t *supersteps,
                                     int64_t *host_checks) {
    if (!g) return fail(FALCON_ERR_INVALID_ARG, "graph is NULL");
    if (!g->comm) return fail(FALCON_ERR_UNSUPPORTED, "not a partitioned graph");
    if (exchange_mode) *exchange_mode = (int32_t)g->last_mode;
    if (supersteps) *supersteps = g->last_rounds;
    if (host_checks) *host_checks = g->last_host_checks;
    return FALCON_OK;
}

falcon_status_t graph_owned_range(const falcon_graph_t *g, int64_t *lo, int64_t *hi) {
    if (!g) return fail(FALCON_ERR_INVALID_ARG, "graph is NULL");
    if (lo) *lo = g->comm ? g->lo : 0;
    if (hi) *hi = g->comm ? g->hi : g->n;
    return FALCON_OK;
}

falcon_status_t falcon_partition(int64_t n, const uint32_t *row_off, int nparts, int64_t *bounds) {
    if (n < 1 || !row_off || !bounds || nparts < 1) return fail(FALCON_ERR_INVALID_ARG, "bad partition arguments");
    partition_bounds(n, row_off, nparts, bounds);
    return FALCON_OK;
}

falcon_status_t falcon_comm_unique_id(void *id128) {
    if (!id128) return fail(FALCON_ERR_INVALID_ARG, "id is NULL");
    NcclApi *nc = nccl_api();
    if (!nc) return fail(FALCON_ERR_COMM, "libnccl.so.2 could not be loaded");
    ncclUniqueId id;
    NC(nc->GetUniqueId(&id));
    memcpy(id128, &id, sizeof id);
    return FALCON_OK;
}

falcon_status_t falcon_comm_loopback_id(int nranks, void *id128) {
    if (!id128 || nranks < 1 || nranks > 64) return fail(FALCON_ERR_INVALID_ARG, "nranks must be in [1, 64]");
    LbWorld *w = new (std::nothrow) LbWorld(nranks);
    if (!w) return fail(FALCON_ERR_NO_MEMORY, "host allocation failed");
    memset(id128, 0, NCCL_UNIQUE_ID_BYTES);
    memcpy(id128, LB_MAGIC, 8);
    memcpy(static_cast<char *>(id128) + 8, &w, sizeof w);
    return FALCON_OK;
}

falcon_status_t falcon_comm_init(int nranks, int rank, const void *id128, int device, falcon_comm_t **out) {
    if (!out || !id128 || nranks < 1 || rank < 0 || rank >= nranks) return fail(FALCON_ERR_INVALID_ARG, "bad comm arguments");
    *out = nullptr;
    const bool loop = memcmp(id128, LB_MAGIC, 8) == 0;
    NcclApi *nc = loop ? loopback_api() : nccl_api();
    if (!nc) return fail(FALCON_ERR_COMM, "libnccl.so.2 could not be loaded");
    CU(cudaSetDevice(device));
    falcon_comm *cm = new (std::nothrow) falcon_comm();
    if (!cm) return fail(FALCON_ERR_NO_MEMORY, "host allocation failed");
    cm->nranks = nranks; cm->rank = rank; cm->device = device;
    cm->api = nc; cm->loopback = loop;
    ncclUniqueId id;
    memcpy(&id, id128, sizeof id);
    ncclResult_t r = nc->CommInitRank(&cm->nccl, nranks, id, rank);
    if (r != ncclSuccess) {
        delete cm;
        return fail(FALCON_ERR_COMM, "ncclCommInitRank: %s", nc->GetErrorString ? nc->GetErrorString(r) : "?");
    }
    *out = cm;
    return FALCON_OK;
}

falcon_status_t falcon_comm_init_simulated(int nparts, falcon_comm_t **out) {
    if (!out || nparts < 1 || nparts > 64) return fail(FALCON_ERR_INVALID_ARG, "nparts must be in [1, 64]");
    falcon_comm *cm = new (std::nothrow) falcon_comm();
    if (!cm) return fail(FALCON_ERR_NO_MEMORY, "host allocation failed");
    cm->simulated = nparts;
    cm->nranks = 1;
    *out = cm;
    return FALCON_OK;
}

falcon_status_t falcon_comm_free(falcon_comm_t *cm) {
    if (!cm) return FALCON_OK;
    if (cm->nccl && cm->api && cm->api->CommDestroy) cm->api->CommDestroy(cm->nccl);
    delete cm;
    return FALCON_OK;
}

falcon_status_t graph_info(const falcon_graph_t *g, int64_t *n, int64_t *m) {
    if (!g) return fail(FALCON_ERR_INVALID_ARG, "graph is NULL");
    if (n) *n = g->n;
    if (m) *m = g->m;
    return FALCON_OK;
}

falcon_status_t falcon_sssp(falcon_graph_t *g, uint32_t source, falcon_style_t style, int32_t *dist_out,
                            falcon_stats_t *stats) {
    NvtxRange r(NVTX_SSSP[(unsigned)style & 3u]);
    return run(g, SSSP, source, (int)style, dist_out, stats);
}

falcon_status_t falcon_bfs(falcon_graph_t *g, uint32_t source, falcon_style_t style, int32_t *level_out,
                           falcon_stats_t *stats) {
    NvtxRange r(NVTX_BFS[(unsigned)style & 3u]);
    return run(g, BFS, source, (int)style, level_out, stats);
}

falcon_status_t falcon_cc(falcon_graph_t *g, falcon_style_t style, int32_t *label_out, falcon_stats_t *stats) {
    NvtxRange r(NVTX_CC[(unsigned)style & 3u]);
    return run(g, CC, 0, (int)style, label_out, stats);
}

falcon_status_t falcon_mst(falcon_graph_t *g, falcon_style_t style, int64_t *total_weight, int64_t *forest_edges,
                           int32_t *label_out, falcon_stats_t *stats) {
    NvtxRange r("falcon_mst");
    return run_mst(g, (int)style, total_weight, forest_edges, label_out, stats);
}

falcon_status_t falcon_set_delta(falcon_graph_t *g, int32_t delta) {
    if (!g) return fail(FALCON_ERR_INVALID_ARG, "graph is NULL");
    if (delta < 0) return fail(FALCON_ERR_INVALID_ARG, "delta must be >= 0 (0 = auto)");
    g->delta = delta;
    return FALCON_OK;
}

falcon_status_t falcon_set_option(falcon_graph_t *g, const char *name, int64_t value) {
    if (!g || !name) return fail(FALCON_ERR_INVALID_ARG, "graph or option name is NULL");
    if ((value < 0 && !(value == -1 && !strcmp(name, "bfs_unit"))) || value > 0xffffffffll)
        return fail(FALCON_ERR_INVALID_ARG, "option value out of range");
    std::vector<falcon_graph *> targets;
    if (g->comm) targets = g->parts; else targets.push_back(g);
    for (falcon_graph *t : targets) {
        if (!strcmp(name, "block_bytes")) {
            if (t->parent || t->nviews)
                return fail(FALCON_ERR_UNSUPPORTED, "block_bytes of a graph shared with views (the layout is shared)");
            if (t->stream) cudaStreamSynchronize(t->stream);
            dfree(t->rowb); dfree(t->cwb); dfree(t->srcb); dfree(t->chunkb);
            t->rowb = nullptr; t->cwb = nullptr; t->srcb = nullptr; t->chunkb = nullptr; t->nblk = 1; t->bsz = 0;
            t->blk_bytes = (size_t)value;
        } else if (!strcmp(name, "dense_div")) {
            t->dense_div = (uint32_t)value;
        } else if (!strcmp(name, "block_div")) {
            t->blk_div = (uint32_t)value;
        } else if (!strcmp(name, "exchange")) {
            if (value > 3) return fail(FALCON_ERR_INVALID_ARG, "exchange: 0 auto, 1 dense, 2 sparse, 3 fused");
            g->exchange = (uint32_t)value;
        } else if (!strcmp(name, "wl_noq")) {
            t->wl_noq = (uint32_t)(value != 0);
        } else if (!strcmp(name, "dl_noq")) {
            t->dl_noq = (uint32_t)(value != 0);
        } else if (!strcmp(name, "split_div")) {
            t->split_div = (uint32_t)value;
        } else if (!strcmp(name, "local")) {
            t->local_tiles = (uint32_t)value;
        } else if (!strcmp(name, "bfs_unit")) {
            if (value < -1 || value > 1) return fail(FALCON_ERR_INVALID_ARG, "bfs_unit: -1 auto, 0 off, 1 on");
            t->bfs_unit = (int32_t)value;
        } else if (!strcmp(name, "local_max")) {
            t->local_max = (uint32_t)std::min<int64_t>(value, 0xffffffffll);
        } else if (!strcmp(name, "wl_local")) {
            t->wl_local_tiles = (uint32_t)value;
        } else if (!strcmp(name, "wl_local_max")) {
            t->wl_local_max = (uint32_t)std::min<int64_t>(value, 0xffffffffll);
        } else if (!strcmp(name, "pull_div")) {
            t->pull_div = (uint32_t)value;
        } else if (!strcmp(name, "bfs_lazy_div")) {
            t->lazy_div = (uint32_t)value;
        } else if (!strcmp(name, "cta_thr")) {
            t->cta_thr = (uint32_t)value;
        } else if (!strcmp(name, "skip_now")) {
            t->skip_now = (uint32_t)value;
        } else if (!strcmp(name, "bfs_wl_pull")) {
            t->wl_pull = (uint32_t)value;
        } else if (!strcmp(name, "pull_rule")) {
            t->pull_rule = (uint32_t)value;
        } else if (!strcmp(name, "persist")) {
            if (value && t->grid_persist <= 0) return fail(FALCON_ERR_UNSUPPORTED, "cooperative launch unavailable");
            t->persist = value != 0;
        } else if (!strcmp(name, "persist_max")) {
            t->persist_max = (uint32_t)value;
        } else {
            return fail(FALCON_ERR_UNSUPPORTED, "unknown option '%s'", name);
        }
        drop_graphs(t);
    }
    return FALCON_OK;
}

falcon_status_t falcon_set_profiling(falcon_graph_t *g, int enable) {
    if (!g) return fail(FALCON_ERR_INVALID_ARG, "graph is NULL");
    g->profiling = enable != 0;
    return FALCON_OK;
}

const char *falcon_last_error(void) { return g_last_error.c_str(); }

const char *falcon_version(void) { return "falcon-b200 0.1 (sm_100a)"; }

}  // extern "C"
