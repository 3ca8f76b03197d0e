/*
 * oracle/oracle.c -- plain, slow, obviously-correct CPU oracle.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (paper_1903_01665_b200/) never links, imports or calls it, and
 * it shares no code, header or constant generator with the CUDA path.
 *
 * What the method computes (Alg. "SSSP: iterating over
 * Points in Falcon"; §2): MIN(t.dist, p.dist + w, changed)
 * applied over all arcs p->t until nothing changes, from dist[source]=0 and
 * dist=MAX_INT elsewhere.  With non-negative integer weights that fixpoint is
 * exactly (up to nothing: integers) the plain definition
 *        dist[v] = min over directed paths source ~> v of the sum of weights,
 * so the oracle writes that definition out with textbook algorithms:
 *
 *   oracle_sssp : Dijkstra with a binary heap (lazy deletion), int64 sums.
 *   oracle_bfs  : FIFO-queue BFS -- the level of PAPER.md:1302-1329
 *                 (Alg. "BFS Algorithm in Falcon for CPU") is the hop count.
 *   oracle_cc   : union-find over all arcs (weak components), label = minimum
 *                 vertex id in the component (SPEC.md:452 min-label
 *                 convention; reading R6).
 *   oracle_mst  : Kruskal over the undirected view -> total weight of a
 *                 minimum spanning forest (§8(f) row 4).
 *
 * Conventions (DESIGN.md §2 readings): INF = 2147483647 = MAX_INT
 * (PAPER.md:1679); weights must be >= 0; a finite
 * distance >= INF is reported as overflow (return 2).  Single-threaded.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_INF 2147483647LL

/* ---------------- binary min-heap of (key, vertex) ---------------- */
typedef struct { int64_t key; uint32_t v; } item_t;
typedef struct { item_t *a; uint64_t len, cap; } heap_t;

static int heap_push(heap_t *h, int64_t key, uint32_t v) {
    if (h->len == h->cap) {
        uint64_t nc = h->cap ? 2 * h->cap : 1024;
        item_t *na = (item_t *)realloc(h->a, nc * sizeof(item_t));
        if (!na) return -1;
        h->a = na; h->cap = nc;
    }
    uint64_t i = h->len++;
    while (i > 0) {                       /* sift up */
        uint64_t p = (i - 1) / 2;
        if (h->a[p].key <= key) break;
        h->a[i] = h->a[p]; i = p;
    }
    h->a[i].key = key; h->a[i].v = v;
    return 0;
}

static item_t heap_pop(heap_t *h) {
    item_t top = h->a[0];
    item_t last = h->a[--h->len];
    uint64_t i = 0;
    for (;;) {                            /* sift down */
        uint64_t l = 2 * i + 1, r = l + 1, s = i;
        int64_t sk = last.key;
        if (l < h->len && h->a[l].key < sk) { s = l; sk = h->a[l].key; }
        if (r < h->len && h->a[r].key < sk) { s = r; }
        if (s == i) break;
        h->a[i] = h->a[s]; i = s;
    }
    if (h->len > 0) h->a[i] = last;
    return top;
}

/* SSSP by Dijkstra.  Returns 0 ok, 1 bad argument / negative weight,
 * 2 overflow (a finite distance would be >= INF), 3 out of memory.
 * w == NULL means every weight is 1. */
int oracle_sssp(int64_t n, const uint32_t *row_off, const uint32_t *col, const int32_t *w,
                uint32_t source, int32_t *dist) {
    if (n <= 0 || (int64_t)source >= n) return 1;
    int64_t *d = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    unsigned char *done = (unsigned char *)calloc((size_t)n, 1);
    if (!d || !done) { free(d); free(done); return 3; }
    for (int64_t v = 0; v < n; v++) d[v] = INT64_MAX;
    heap_t h = {0, 0, 0};
    d[source] = 0;
    int rc = 0;
    if (heap_push(&h, 0, source)) rc = 3;
    while (rc == 0 && h.len > 0) {
        item_t it = heap_pop(&h);
        uint32_t u = it.v;
        if (done[u] || it.key != d[u]) continue;      /* stale entry */
        done[u] = 1;
        for (uint32_t e = row_off[u]; e < row_off[u + 1]; e++) {
            int64_t wt = w ? (int64_t)w[e] : 1;
            if (wt < 0) { rc = 1; break; }
            uint32_t v = col[e];
            int64_t cand = d[u] + wt;
            if (cand < d[v]) {
                d[v] = cand;
                if (heap_push(&h, cand, v)) { rc = 3; break; }
            }
        }
    }
    if (rc == 0) {
        for (int64_t v = 0; v < n; v++) {
            if (d[v] == INT64_MAX) dist[v] = (int32_t)ORACLE_INF;
            else if (d[v] >= ORACLE_INF) { rc = 2; dist[v] = (int32_t)ORACLE_INF; }
            else dist[v] = (int32_t)d[v];
        }
    }
    free(h.a); free(d); free(done);
    return rc;
}

/* BFS levels (hop distance) by a FIFO queue.  Returns 0 ok, 1 bad arg, 3 OOM. */
int oracle_bfs(int64_t n, const uint32_t *row_off, const uint32_t *col, uint32_t source, int32_t *level) {
    if (n <= 0 || (int64_t)source >= n) return 1;
    uint32_t *q = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
    if (!q) return 3;
    for (int64_t v = 0; v < n; v++) level[v] = (int32_t)ORACLE_INF;
    int64_t head = 0, tail = 0;
    level[source] = 0;
    q[tail++] = source;
    while (head < tail) {
        uint32_t u = q[head++];
        for (uint32_t e = row_off[u]; e < row_off[u + 1]; e++) {
            uint32_t v = col[e];
            if (level[v] == (int32_t)ORACLE_INF) {
                level[v] = level[u] + 1;
                q[tail++] = v;
            }
        }
    }
    free(q);
    return 0;
}

/* Union-find with union by size and path halving. */
static uint32_t uf_find(uint32_t *parent, uint32_t x) {
    while (parent[x] != x) {
        parent[x] = parent[parent[x]];
        x = parent[x];
    }
    return x;
}

/* Weakly connected components, label = min vertex id of the component.
 * Returns 0 ok, 3 OOM.  n == 0 is allowed. */
int oracle_cc(int64_t n, const uint32_t *row_off, const uint32_t *col, int32_t *label) {
    if (n < 0) return 1;
    if (n == 0) return 0;
    uint32_t *parent = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
    uint32_t *size = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
    int64_t *minid = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    if (!parent || !size || !minid) { free(parent); free(size); free(minid); return 3; }
    for (int64_t v = 0; v < n; v++) { parent[v] = (uint32_t)v; size[v] = 1; minid[v] = -1; }
    for (int64_t u = 0; u < n; u++) {
        for (uint32_t e = row_off[u]; e < row_off[u + 1]; e++) {
            uint32_t a = uf_find(parent, (uint32_t)u), b = uf_find(parent, col[e]);
            if (a == b) continue;
            if (size[a] < size[b]) { uint32_t t = a; a = b; b = t; }
            parent[b] = a; size[a] += size[b];
        }
    }
    for (int64_t v = 0; v < n; v++) {              /* ascending: first member seen is the min id */
        uint32_t r = uf_find(parent, (uint32_t)v);
        if (minid[r] < 0) minid[r] = v;
        label[v] = (int32_t)minid[r];
    }
    free(parent); free(size); free(minid);
    return 0;
}

/* ---------------- minimum spanning forest ----------------
 * The paper's fourth algorithm ("Minimum Spanning Tree computation
 * (MST)", Table 2 MST column); "MST total weight == Kruskal
 * oracle".  Every arc u->v is the undirected edge {u, v} (the graph is a
 * directed multigraph; SPEC.md:571 duplicates tolerated), so the result is a
 * minimum spanning forest: one minimum spanning tree per weak component.
 * Kruskal (1956): arcs in ascending weight order (ties by arc index), an arc
 * joins the forest iff its endpoints lie in different trees (union-find).
 *   *total  = sum of the weights of the joined arcs -- the same for every
 *             minimum spanning forest, whatever the order among equal weights;
 *   *nedges = number of joined arcs = n - #components;
 *   label   = (nullable) min vertex id of the tree (= the CC label).
 * w == NULL means every weight is 1.  Returns 0 ok, 1 bad argument / negative
 * weight, 3 OOM. */
static const int32_t *g_mst_w;
static int mst_cmp(const void *a, const void *b) {
    const uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
    const int32_t wx = g_mst_w ? g_mst_w[x] : 1, wy = g_mst_w ? g_mst_w[y] : 1;
    if (wx != wy) return wx < wy ? -1 : 1;
    return x < y ? -1 : (x > y ? 1 : 0);
}

int oracle_mst(int64_t n, const uint32_t *row_off, const uint32_t *col, const int32_t *w, int64_t *total,
               int64_t *nedges, int32_t *label) {
    if (n < 0 || !row_off || !total || !nedges) return 1;
    *total = 0; *nedges = 0;
    if (n == 0) return 0;
    const uint64_t m = row_off[n];
    if (w)
        for (uint64_t e = 0; e < m; e++)
            if (w[e] < 0) return 1;
    uint32_t *src = (uint32_t *)malloc((m ? m : 1) * sizeof(uint32_t));
    uint32_t *order = (uint32_t *)malloc((m ? m : 1) * sizeof(uint32_t));
    uint32_t *parent = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
    uint32_t *size = (uint32_t *)malloc((size_t)n * sizeof(uint32_t));
    int64_t *minid = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    if (!src || !order || !parent || !size || !minid) {
        free(src); free(order); free(parent); free(size); free(minid);
        return 3;
    }
    for (int64_t u = 0; u < n; u++)
        for (uint32_t e = row_off[u]; e < row_off[u + 1]; e++) src[e] = (uint32_t)u;
    for (uint64_t e = 0; e < m; e++) order[e] = (uint32_t)e;
    g_mst_w = w;
    qsort(order, m, sizeof(uint32_t), mst_cmp);
    for (int64_t v = 0; v < n; v++) { parent[v] = (uint32_t)v; size[v] = 1; minid[v] = -1; }
    for (uint64_t i = 0; i < m; i++) {
        const uint32_t e = order[i];
        uint32_t a = uf_find(parent, src[e]), b = uf_find(parent, col[e]);
        if (a == b) continue;                      /* would close a cycle (or a self loop) */
        if (size[a] < size[b]) { uint32_t t = a; a = b; b = t; }
        parent[b] = a; size[a] += size[b];
        *total += w ? w[e] : 1;
        *nedges += 1;
    }
    if (label) {
        for (int64_t v = 0; v < n; v++) {
            uint32_t r = uf_find(parent, (uint32_t)v);
            if (minid[r] < 0) minid[r] = v;
            label[v] = (int32_t)minid[r];
        }
    }
    free(src); free(order); free(parent); free(size); free(minid);
    return 0;
}
