/*
 * falcon.h -- C ABI of the B200-native fixpoint min-relaxation library
 * (SSSP / BFS / connected components) after arXiv 1903.01665 ("adaptive
 * Falcon").  Plain C types only: no torch, no CUDA types in the signatures
 * (streams are passed as void*).
 *
 * The operation (Alg. "SSSP: iterating over Points in
 * Falcon", Alg. "SSSP: iterating over Edges";
 * PAPER.md:1727-1730 §2): starting from dist[source] = 0 and dist = MAX_INT
 * elsewhere, apply  MIN(t.dist, p.dist + weight(p->t), changed)  to arcs p->t
 * until no value changes.  BFS is the level-synchronous variant of
 * PAPER.md:1302-1329 (Alg. "BFS Algorithm in Falcon for CPU"); CC is the
 * "propagation based" component labelling named at PAPER.md:7, 73.
 *
 * The three processing styles are the paper's vertex-based, edge-based and
 * worklist-based codes (§3.1, 1567-1571 §3.3), selected at
 * run time instead of compile time.  All styles return
 * bit-identical results: each output is the unique least fixpoint.
 *
 * Common conventions
 *  - Every call is synchronous: it returns with its outputs complete.  Work is
 *    issued on the stream given at load time (falcon_load_opts_t.cuda_stream,
 *    a cudaStream_t passed as void*), or on a stream the graph owns.
 *  - Pointers marked (host|device) may be either; the library detects which
 *    with cudaPointerGetAttributes and copies accordingly.  Inputs are only
 *    borrowed for the duration of the call.  Outputs are caller-allocated.
 *  - Errors are returned as falcon_status_t, never thrown; a thread-local
 *    message is available from falcon_last_error().  After a non-OK status the
 *    outputs are unspecified; the graph stays usable except after
 *    FALCON_ERR_CUDA.
 *  - Not thread-safe per graph: do not call two algorithms on the same
 *    falcon_graph_t concurrently (they share the graph's scratch buffers).
 */
#ifndef FALCON_H
#define FALCON_H

#include <stdint.h>

#if defined(__GNUC__)
#define FALCON_API __attribute__((visibility("default")))
#else
#define FALCON_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* INF = MAX_INT of PAPER.md:1679 (SSSP) / the BFS "infinity" of PAPER.md:1318,
 * unified as INT32_MAX.  Unreachable vertices report it. */
#define FALCON_INF 2147483647

typedef enum {
    FALCON_STYLE_VERTEX = 0,   /* topology-driven over CSR rows   */
    FALCON_STYLE_EDGE = 1,     /* topology-driven over COO arcs   */
    FALCON_STYLE_WORKLIST = 2, /* data-driven over a frontier queue */
    FALCON_STYLE_DELTA = 3     /* SSSP only: Δ-stepping bucketed worklist (near queue + far set;
                                  PAPER.md:454).  Same result. */
} falcon_style_t;

typedef enum {
    FALCON_OK = 0,
    FALCON_ERR_INVALID_ARG = 1,   /* NULL pointer, n < 1, n >= 2^31, m >= 2^32, bad style      */
    FALCON_ERR_OUT_OF_RANGE = 2,  /* row_off not 0..m nondecreasing, col >= n, w < 0, src >= n */
    FALCON_ERR_NO_MEMORY = 3,     /* device allocation failed                                  */
    FALCON_ERR_CUDA = 4,          /* any other CUDA runtime error (graph may be unusable)      */
    FALCON_ERR_OVERFLOW = 5,      /* SSSP: some vertex's shortest distance is finite but
                                     >= FALCON_INF (decided on the final distances, so the status
                                     never depends on the relaxation schedule; R3)    */
    FALCON_ERR_NOT_CONVERGED = 6, /* iteration cap (n + 2 rounds; DELTA 10 n)      */
    FALCON_ERR_COMM = 7,          /* reserved: multi-GPU communication failure                 */
    FALCON_ERR_UNSUPPORTED = 8    /* option not supported by this build                        */
} falcon_status_t;

typedef struct falcon_graph falcon_graph_t; /* opaque; owns its device memory */
typedef struct falcon_comm falcon_comm_t;   /* opaque; multi-GPU communicator (NULL = single GPU) */

/* graph_load_csr options (pass NULL for defaults). */
#define FALCON_LOAD_BUILD_COO 0x1u      /* build the COO src[] array now (else lazily on first EDGE call) */
#define FALCON_LOAD_BUILD_REVERSE 0x2u  /* build the reverse (in-arc) CSR now (else lazily on the first BFS
                                           VERTEX / CC WORKLIST call) */
/* Partitioned graphs (opts.comm != NULL) only -- per-GPU graph copies of the
 * paper's multi-GPU runs (§3.4) without the full graph on
 * every rank: */
#define FALCON_LOAD_SLICE 0x4u   /* this rank passes ONLY its own rows: n = rows of the slice, m = their arcs,
                                    row_off = the slice's offsets (row_off[0] == 0, row_off[n] == m), col =
                                    GLOBAL target ids.  The ranks' slices, in rank order, are the graph: rank
                                    r owns the vertices after those of ranks < r (all-gathered at load; the
                                    global n is their total).  Needs a rank communicator (NCCL or loopback),
                                    not a simulated one (UNSUPPORTED).  Validated on the device against the
                                    global n -- no full-graph host copy. */
#define FALCON_LOAD_GATHER 0x8u  /* every algorithm call writes the FULL n-length output on every rank (an
                                    all-gather of the owned slices).  Default for rank communicators: each
                                    rank receives only its owned slice [lo, hi) (graph_owned_range), an
                                    int32[hi - lo] buffer.  Simulated graphs always return the full array. */

typedef struct {
    int device;          /* CUDA device ordinal; -1 = current device                 */
    void *cuda_stream;   /* cudaStream_t to issue work on; NULL = a stream owned by the graph */
    uint32_t flags;      /* FALCON_LOAD_* bits                                       */
    falcon_comm_t *comm; /* NULL = single GPU; else a 1-D vertex-partitioned graph    */
} falcon_load_opts_t;

/* Per-call statistics (all counters are device-side totals for the call). */
typedef struct {
    int64_t iterations;         /* fixpoint rounds executed (BFS: levels + 1)              */
    int64_t vertices_processed; /* active vertices / frontier items expanded                */
    int64_t edges_relaxed;      /* arcs on which MIN was evaluated                          */
    int64_t updates;            /* successful MIN updates (value strictly decreased)        */
    int64_t kernel_launches;    /* library kernels launched for the call                   */
    double ms;                  /* device time from init to result (CUDA events), excl. D2H */
    double relax_ms;            /* profiling mode only: summed relax-kernel time, else -1  */
    int64_t relax_launches;     /* profiling mode only: relax-kernel launches, else 0      */
} falcon_stats_t;

/* Load a graph in CSR form (§3.1: CSR for vertex-based,
 * an edge list for edge-based code; SPEC.md:408-413 GraphStore invariants).
 *   n        vertices, 1 <= n < 2^31
 *   m        arcs, 0 <= m < 2^32
 *   row_off  (host|device) uint32[n+1]: row_off[0]==0, nondecreasing, row_off[n]==m
 *   col      (host|device) uint32[m]: arc targets, each < n
 *   w        (host|device) int32[m] arc weights >= 0, or NULL = every weight 1
 *   opts     NULL or options above
 *   out      receives the new graph handle (owned by the caller; free with graph_free)
 * Copies everything into library-owned, 16-byte aligned device arrays.
 * Errors: INVALID_ARG, OUT_OF_RANGE (validated on the device), NO_MEMORY, CUDA. */
FALCON_API falcon_status_t graph_load_csr(int64_t n, int64_t m, const uint32_t *row_off, const uint32_t *col,
                               const int32_t *w, const falcon_load_opts_t *opts, falcon_graph_t **out);

/* ---- multi-GPU: 1-D vertex partition ----
 * Vertices are split into contiguous ranges; part q stores the CSR rows of
 * its range.  Either every rank passes the FULL CSR (ranges of ~m/P arcs are
 * chosen by binary search on row_off; each rank keeps only its rows) or each
 * rank passes only its own rows (FALCON_LOAD_SLICE).  All ranks then call the
 * algorithms collectively, in the same order.  Per superstep the boundary
 * values travel by the "exchange" option (falcon_set_option): by default the
 * relax kernel itself writes every remote improvement into its owner's arrays
 * over peer memory (NVLink via CUDA IPC) -- fused, no exchange step -- else a
 * grouped ncclReduce(MIN) to the owners (dense) or (vertex, value) pairs
 * (sparse); termination is an ncclAllReduce(SUM) of the round's `changed`
 * flag, and the host checks for the fixpoint once every 4 supersteps.  Output:
 * the owned slice per rank, or the full array with FALCON_LOAD_GATHER.
 * Results equal the single-GPU ones.  BFS runs as unit-weight SSSP; CC hooks
 * on a replicated label array (ncclAllReduce(MIN) per round).  The processing
 * style is ignored (every part runs the VERTEX round). */

/* Partition boundaries: bounds[q] .. bounds[q+1] is part q's vertex range,
 * chosen so each part owns ~m/nparts arcs (binary search on row_off).
 * row_off: HOST uint32[n+1].  bounds: HOST int64[nparts+1].  No GPU needed. */
FALCON_API falcon_status_t falcon_partition(int64_t n, const uint32_t *row_off, int nparts, int64_t *bounds);

/* 128-byte NCCL unique id for falcon_comm_init (call on one rank, broadcast
 * it out of band, e.g. with torch.distributed).  Errors: COMM (no NCCL). */
FALCON_API falcon_status_t falcon_comm_unique_id(void *id128);

/* One rank of an nranks-wide communicator on `device` (one process per GPU;
 * NCCL over NVLink / NVSwitch), or of a loopback world when id128 comes from
 * falcon_comm_loopback_id.  Errors: INVALID_ARG, COMM, CUDA. */
FALCON_API falcon_status_t falcon_comm_init(int nranks, int rank, const void *id128, int device, falcon_comm_t **out);

/* A 128-byte id for an in-process LOOPBACK communicator of nranks ranks: pass
 * it to falcon_comm_init from nranks host threads of THIS process (any device,
 * typically the same one).  The ranks then run exactly the code path of NCCL
 * ranks -- slice loading, exchanges, termination, owned-slice output -- with
 * every NCCL call served in-process (device copies, host barriers): how the
 * per-rank multi-GPU path is tested on a one-GPU box (NCCL refuses two ranks
 * on one device).  Free each rank's communicator with falcon_comm_free.
 * Errors: INVALID_ARG (nranks not in [1, 64]), NO_MEMORY. */
FALCON_API falcon_status_t falcon_comm_loopback_id(int nranks, void *id128);

/* A simulated communicator: nparts partitions on the current device of ONE
 * process, exchanged by device kernels (same partition, relax, apply and
 * termination code; used to test the partitioned algorithm on one GPU). */
FALCON_API falcon_status_t falcon_comm_init_simulated(int nparts, falcon_comm_t **out);

FALCON_API falcon_status_t falcon_comm_free(falcon_comm_t *comm);

/* Vertex range [lo, hi) owned by this rank ([0, n) for a single-GPU or a
 * simulated graph); the output of a rank's call is this slice unless the
 * graph was loaded with FALCON_LOAD_GATHER. */
FALCON_API falcon_status_t graph_owned_range(const falcon_graph_t *g, int64_t *lo, int64_t *hi);

/* Bytes the last call on a partitioned graph moved in its boundary exchanges
 * (dense reduce-scatter rounds: 4 bytes per exchanged vertex; sparse rounds:
 * 8 bytes per (vertex, value) pair; fused rounds: 8 bytes -- a RED.MIN and a
 * bitmap RED.OR -- per remote improvement; CC: the 4n-byte label all-reduce
 * per round; this rank's sends, or all parts when simulated).  0 for a
 * single-GPU graph. */
FALCON_API falcon_status_t graph_exchange_bytes(const falcon_graph_t *g, int64_t *bytes);

/* The last call on a partitioned graph: *exchange_mode = the exchange its
 * supersteps used (1 dense, 2 sparse, 3 fused), *supersteps = rounds run,
 * *host_checks = host round trips of the fixpoint loop (one per 4 supersteps;
 * the sparse exchange adds its per-superstep count syncs).  Any pointer may be
 * NULL.  Errors: INVALID_ARG (NULL g), UNSUPPORTED (not partitioned). */
FALCON_API falcon_status_t graph_partition_info(const falcon_graph_t *g, int32_t *exchange_mode, int64_t *supersteps,
                                                int64_t *host_checks);

/* Release the graph's device memory (to the library's device-memory cache,
 * which later loads reuse; a failed allocation releases the cache).  NULL is a
 * no-op.  Errors: INVALID_ARG if views created by graph_share are still live. */
FALCON_API falcon_status_t graph_free(falcon_graph_t *g);

/* A view of g for concurrent calls: it shares g's read-only graph arrays
 * (CSR, COO, chunk ranges, blocked and reverse layouts -- all built now, on g)
 * and owns its own scratch (value array, bitmaps, queues, control block,
 * stream, cached CUDA graphs).  Calls on g and on each of its views may then
 * run at the same time, from different host threads or through
 * falcon_run_many -- the paper's concurrent BFS/SSSP kernels
 * (PAPER.md:1040-1064, 1137-1142 §"Synchronous vs asynchronous").  opts:
 * nullable; only cuda_stream is used (NULL = a stream the view owns).  A view
 * of a view shares the root graph.  Free views (graph_free) before g.
 * Errors: INVALID_ARG (NULL), UNSUPPORTED (partitioned g), NO_MEMORY, CUDA. */
FALCON_API falcon_status_t graph_share(falcon_graph_t *g, const falcon_load_opts_t *opts, falcon_graph_t **out);

typedef enum { FALCON_ALGO_SSSP = 0, FALCON_ALGO_BFS = 1, FALCON_ALGO_CC = 2 } falcon_algo_t;

typedef struct {
    falcon_algo_t algo;
    falcon_style_t style;
    uint32_t source; /* ignored for CC */
} falcon_job_t;

/* Run njobs calls concurrently: job i runs on graphs[i] (distinct handles --
 * a graph and its views) and writes outs[i] (host|device int32[n]); every job
 * is launched on its handle's stream before any is waited on.  stats: NULL or
 * falcon_stats_t[njobs].  Returns when all jobs are complete; on error the
 * first failing job's status (all launched jobs are still completed).
 * Results equal those of the one-at-a-time calls.
 * Errors: INVALID_ARG (NULL arrays, repeated handle, unknown algo/style,
 * source >= n), UNSUPPORTED (partitioned graph), plus the per-call statuses. */
FALCON_API falcon_status_t falcon_run_many(int njobs, falcon_graph_t *const *graphs, const falcon_job_t *jobs,
                                           int32_t *const *outs, falcon_stats_t *stats);

/* Return the device memory the library keeps cached for reuse (blocks of
 * freed graphs and per-call staging) to the CUDA driver; *released_bytes
 * (nullable) receives the amount.  Live graphs are not affected. */
FALCON_API falcon_status_t falcon_trim_memory(int64_t *released_bytes);

/* Query vertex / arc counts of a loaded graph. */
FALCON_API falcon_status_t graph_info(const falcon_graph_t *g, int64_t *n, int64_t *m);

/* Single-source shortest paths: dist_out[v] = min over directed paths
 * source ~> v of the sum of weights, FALCON_INF if unreachable
 * (PAPER.md:1727-1730).  dist_out: (host|device) int32[n].  stats: nullable.
 * Errors: INVALID_ARG (source >= n, bad style), OVERFLOW, NOT_CONVERGED, CUDA. */
FALCON_API falcon_status_t falcon_sssp(falcon_graph_t *g, uint32_t source, falcon_style_t style, int32_t *dist_out,
                            falcon_stats_t *stats);

/* Breadth-first levels: level_out[v] = fewest arcs on a directed path
 * source ~> v, FALCON_INF if unreachable.  Weights are
 * ignored.  level_out: (host|device) int32[n]. */
FALCON_API falcon_status_t falcon_bfs(falcon_graph_t *g, uint32_t source, falcon_style_t style, int32_t *level_out,
                           falcon_stats_t *stats);

/* Connected components of the undirected view (weak components): label_out[v]
 * = smallest vertex id in v's component (min-label convention
 * SPEC.md:452).  Weights and arc direction are ignored.
 * label_out: (host|device) int32[n]. */
FALCON_API falcon_status_t falcon_cc(falcon_graph_t *g, falcon_style_t style, int32_t *label_out, falcon_stats_t *stats);

/* Minimum spanning forest of the undirected view (every arc u->v is the edge
 * {u, v}; self loops never join, duplicates allowed): *total_weight = the
 * total weight of a minimum spanning tree of every weak component -- the
 * paper's MST (Table 2), checked against Kruskal (SPEC.md:470,
 * 492).  Borůvka rounds: per round every component picks its
 * lightest incident arc (ties by arc index), components hook across their
 * picks, pointer jumping flattens; at most log2(n) + 1 rounds.
 * forest_edges (nullable) = number of forest edges = n - #components;
 * label_out (nullable, host|device int32[n]) = min vertex id of the vertex's
 * tree (= the CC label).  style: VERTEX (CSR rows) or EDGE (COO arcs).
 * Errors: INVALID_ARG (NULL g / total_weight), UNSUPPORTED (other styles,
 * partitioned graph), CUDA. */
FALCON_API falcon_status_t falcon_mst(falcon_graph_t *g, falcon_style_t style, int64_t *total_weight,
                                      int64_t *forest_edges, int32_t *label_out, falcon_stats_t *stats);

/* Bucket width Δ of FALCON_STYLE_DELTA (SSSP): vertices with tentative
 * distance < T are relaxed from the near queue, the others wait in a far set
 * until the near queue is empty and T advances to the next non-empty bucket.
 * delta == 0 (default) = start at max(1, average arc weight)
 * and adapt per bucket (double while rounds are latency-bound, halve while
 * they relax millions of items); delta > 0 is kept fixed.
 * Errors: INVALID_ARG (g NULL or delta < 0). */
FALCON_API falcon_status_t falcon_set_delta(falcon_graph_t *g, int32_t delta);

/* Tuning options of a loaded graph (results never depend on them; they pick
 * the data layout and schedule).  name / value:
 *   "block_bytes"  value-array bytes per destination block of the SSSP arc
 *                  layout (default 64 MiB, env FALCON_BLOCK_MB; 0 = no blocking)
 *   "dense_div"    a round is dense (bitmap-driven, items in vertex order)
 *                  when its frontier exceeds n / dense_div (default 32,
 *                  env FALCON_DENSE_DIV; 0 = never)
 *   "block_div"    an SSSP round walks the blocked layout when its frontier
 *                  exceeds n / block_div (default 8, env FALCON_BLOCK_DIV;
 *                  0 = never)
 *   "pull_div"     BFS VERTEX may run bottom-up (over in-arcs)
 *                  only while the frontier exceeds n / pull_div under rule
 *                  1 / 2 (default 16; 0 = never pull)
 *   "pull_rule"    BFS VERTEX direction per round: 0 = estimated L2 requests
 *                  of a push and a pull round (default),
 *                  1 / 2 = pull iff the frontier exceeds n / pull_div, with
 *                  the word-per-warp / compacted pull form (env
 *                  FALCON_BFS_PULL_RULE)
 *   "cta_thr"      rows longer than this many arcs are expanded by the whole
 *                  CTA instead of one warp (default 1024, env FALCON_CTA_THR;
 *                  0 = warp-level only)
 *   "bfs_wl_pull"  BFS WORKLIST rounds may run bottom-up over the in-arcs
 *                  like VERTEX, by the same per-round cost model (default 1,
 *                  env FALCON_BFS_WL_PULL; 0 = push only)
 *   "skip_now"     SSSP expansion styles: an item whose bit is already set in
 *                  the current round's bitmap (improved again this round, so
 *                  it is expanded next round with its newer value) is not
 *                  expanded now (default 1, env FALCON_SKIP_NOW; 0 = off)
 *   "persist"      queue styles run small rounds in one cooperative kernel (0/1)
 *   "persist_max"  ... while the frontier holds at most this many items
 * Changing an option drops the cached CUDA graphs (and, for block_bytes, the
 * blocked layout); they are rebuilt on the next call.
 *   "exchange"     partitioned graphs: boundary exchange per superstep, 0 = auto
 *                  (fused between ranks that can map each other's memory,
 *                  else dense; dense for simulated parts), 1 = dense
 *                  (grouped ncclReduce(MIN) per owner), 2 = sparse ((vertex,
 *                  value) pairs by ncclSend / ncclRecv; host-synchronised
 *                  per superstep), 3 = fused (relax kernels RED.MIN / RED.OR
 *                  remote targets into their owners' arrays over peer memory;
 *                  NCCL ranks map each other's arrays with CUDA IPC) (env
 *                  FALCON_EXCHANGE)
 *   "wl_noq"       WORKLIST dense rounds mark the next bitmap without claims
 *                  or a queue (default 1, env FALCON_WL_NOQ; 0 = off)
 *   "dl_noq"       the same for DELTA dense rounds (near targets marked, far
 *                  ones parked; default 1, env FALCON_DL_NOQ)
 *   "split_div"    DELTA with auto Δ: a near round that hands on more than
 *                  n / split_div items halves the bucket; items at or beyond
 *                  the new threshold go back to the far set (env
 *                  FALCON_SPLIT_DIV; 0 = never)
 *   "local"        SSSP DELTA sparse rounds: each warp expands the in-bucket
 *                  targets it improved itself, up to this many 32-item tiles
 *                  per round, before handing the rest to the next round's
 *                  queue (env FALCON_LOCAL; 0 = off; default set at load:
 *                  16 when m < 3n, 4 when m < 6n, else 0).  Any relaxation order reaches the
 *                  same fixpoint.
 *   "local_max"    ... only in rounds of at most this many items (env
 *                  FALCON_LOCAL_MAX; default unbounded when m < 3n, else 16384)
 *   "wl_local"     the same for SSSP WORKLIST sparse rounds (env FALCON_WL_LOCAL;
 *                  default set at load: 4 when m < 3n, else 0 = off)
 *   "wl_local_max" ... in rounds of at most this many items (env
 *                  FALCON_WL_LOCAL_MAX; default 262144)
 *   "bfs_unit"     BFS WORKLIST runs as unit-weight Δ-stepping with local
 *                  continuation (same levels): -1 auto (m < 3n and local on;
 *                  the default), 0 off, 1 on (env FALCON_BFS_UNIT)
 * Errors: INVALID_ARG (g/name NULL, value out of range), UNSUPPORTED (unknown
 * name; block_bytes of a graph that has, or is, a view). */
FALCON_API falcon_status_t falcon_set_option(falcon_graph_t *g, const char *name, int64_t value);

/* Profiling mode (off by default): when on, the fixpoint loop is driven from
 * the host and every relax-kernel launch is bracketed by CUDA events, filling
 * falcon_stats_t.relax_ms / relax_launches.  Results are identical. */
FALCON_API falcon_status_t falcon_set_profiling(falcon_graph_t *g, int enable);

/* Thread-local description of the last non-OK status ("" if none). */
FALCON_API const char *falcon_last_error(void);

/* Library version string. */
FALCON_API const char *falcon_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FALCON_H */
