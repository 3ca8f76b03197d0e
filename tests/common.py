"""Test-side helpers: golden fixture loader, brute-force references and
O(m) certificates.  Written independently of both oracle/ and the CUDA path.

Certificates:
  SSSP  d[s]=0, d>=0; feasibility d[v] <= d[u]+w on every arc with d[u]<INF;
        every finite v != s has a tight in-arc; a BFS over tight arcs from s
        reaches every finite v (needed when weights can be 0).
  BFS   level[s]=0; level[v] <= level[u]+1 on every arc; every finite v != s
        has an in-arc from level[v]-1.
  CC    labels equal across every arc; label[v] <= v; label[label[v]] ==
        label[v]; #distinct labels == #weak components (counted here by an
        independent numpy label-propagation-free method: scipy).
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

INF = 2147483647
GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@dataclass
class Golden:
    name: str
    n: int
    src: np.ndarray
    dst: np.ndarray
    w: np.ndarray
    source: int
    expect: dict
    cite: str


def load_golden(fname: str) -> Golden:
    path = os.path.join(GOLDEN_DIR, fname)
    cite, edges, expect = [], [], {}
    n = m = None
    source = 0
    with open(path) as f:
        for line in f:
            line = line.split("#", 1)[0].strip() if not line.startswith("#") else (cite.append(line[1:].strip()) or "")
            if not line:
                continue
            tok = line.split()
            if tok[0] == "p":
                n, m = int(tok[1]), int(tok[2])
            elif tok[0] == "source":
                source = int(tok[1])
            elif tok[0] == "expect":
                expect[tok[1]] = np.array([int(x) for x in tok[2:]], dtype=np.int64)
            else:
                edges.append(tuple(int(x) for x in tok[:3]))
    assert n is not None and len(edges) == m, f"{fname}: header promises {m} arcs, found {len(edges)}"
    e = np.array(edges, dtype=np.int64).reshape(-1, 3)
    return Golden(fname, n, e[:, 0].astype(np.uint32), e[:, 1].astype(np.uint32), e[:, 2].astype(np.int32),
                  source, expect, " ".join(cite))


def golden_files():
    return sorted(f for f in os.listdir(GOLDEN_DIR) if f.endswith(".txt") and f != "table1.txt")


# ------------------------------------------------------------ brute force
def bellman_ford(n, src, dst, w, s):
    """n-1 full rounds over all arcs, int64, exact (Bellman 1958)."""
    d = np.full(n, np.iinfo(np.int64).max, dtype=np.int64)
    d[s] = 0
    big = np.iinfo(np.int64).max
    src = np.asarray(src, np.int64); dst = np.asarray(dst, np.int64); w = np.asarray(w, np.int64)
    for _ in range(max(n - 1, 0)):
        du = d[src]
        ok = du != big
        cand = np.where(ok, du + w, big)
        nd = d.copy()
        np.minimum.at(nd, dst, cand)
        if np.array_equal(nd, d):
            break
        d = nd
    return np.where(d == big, INF, d)


def floyd_warshall_row(n, src, dst, w, s):
    """All-pairs Floyd-Warshall (n <= ~300), return row s."""
    big = np.iinfo(np.int64).max // 4
    D = np.full((n, n), big, dtype=np.int64)
    np.fill_diagonal(D, 0)
    for u, v, wt in zip(np.asarray(src, np.int64), np.asarray(dst, np.int64), np.asarray(w, np.int64)):
        if wt < D[u, v]:
            D[u, v] = wt
    for k in range(n):
        D = np.minimum(D, D[:, k:k + 1] + D[k:k + 1, :])
    row = D[s]
    return np.where(row >= big, INF, row)


def closure_cc(n, src, dst):
    """Weak components by transitive closure of the symmetrised adjacency."""
    A = np.eye(n, dtype=bool)
    A[np.asarray(src, np.int64), np.asarray(dst, np.int64)] = True
    A[np.asarray(dst, np.int64), np.asarray(src, np.int64)] = True
    R = A.copy()
    while True:
        R2 = (R.astype(np.uint8) @ R.astype(np.uint8)) > 0
        if np.array_equal(R2, R):
            break
        R = R2
    return np.array([int(np.argmax(R[v])) for v in range(n)], dtype=np.int64)  # first True = min id


# ------------------------------------------------------------ certificates
def _src_of(row_off):
    deg = np.diff(row_off.astype(np.int64))
    return np.repeat(np.arange(len(row_off) - 1, dtype=np.int64), deg)


def cert_sssp(row_off, col, w, s, d):
    d = np.asarray(d, np.int64)
    n = len(row_off) - 1
    src = _src_of(row_off); dst = col.astype(np.int64)
    wt = np.ones(len(dst), np.int64) if w is None else w.astype(np.int64)
    assert d[s] == 0, "d[s] != 0"
    assert (d >= 0).all(), "negative distance"
    fin_u = d[src] != INF
    assert (d[dst][fin_u] <= d[src][fin_u] + wt[fin_u]).all(), "feasibility violated"
    tight = fin_u & (d[dst] == d[src] + wt)
    has_tight = np.zeros(n, bool)
    has_tight[dst[tight]] = True
    fin = d != INF
    need = fin.copy(); need[s] = False
    assert has_tight[need].all(), "a finite vertex has no tight in-arc"
    # tight-arc reachability from s (zero weights may form tight cycles)
    import scipy.sparse as sp
    from scipy.sparse import csgraph
    T = sp.csr_matrix((np.ones(int(tight.sum()), np.int8), (src[tight], dst[tight])), shape=(n, n))
    seen = np.zeros(n, bool)
    seen[csgraph.breadth_first_order(T, s, directed=True, return_predecessors=False)] = True
    assert (seen == fin).all(), "tight arcs from s do not reach exactly the finite vertices"


def cert_bfs(row_off, col, s, lv):
    lv = np.asarray(lv, np.int64)
    n = len(row_off) - 1
    src = _src_of(row_off); dst = col.astype(np.int64)
    assert lv[s] == 0
    fin_u = lv[src] != INF
    assert (lv[dst][fin_u] <= lv[src][fin_u] + 1).all(), "level jumps by more than 1"
    fin = lv != INF
    has_parent = np.zeros(n, bool)
    par = fin_u & (lv[src] == lv[dst] - 1)
    has_parent[dst[par]] = True
    need = fin.copy(); need[s] = False
    assert has_parent[need].all(), "finite vertex without a parent one level up"
    assert (lv[fin] >= 0).all()


def cert_cc(row_off, col, label, n_components: int):
    lab = np.asarray(label, np.int64)
    n = len(row_off) - 1
    src = _src_of(row_off); dst = col.astype(np.int64)
    assert (lab[src] == lab[dst]).all(), "an arc joins different labels"
    assert (lab <= np.arange(n)).all(), "label > vertex id"
    assert (lab >= 0).all()
    assert (lab[lab] == lab).all(), "label is not its own label"
    assert len(np.unique(lab)) == n_components, "label count != component count"


def scipy_reference(row_off, col, w, s):
    """scipy.sparse.csgraph: (sssp, bfs, cc) with min-combined duplicate arcs."""
    import scipy.sparse as sp
    from scipy.sparse import csgraph
    n = len(row_off) - 1
    src = _src_of(row_off); dst = col.astype(np.int64)
    wt = np.ones(len(dst), np.int64) if w is None else w.astype(np.int64)
    # Min-combine duplicate arcs first: csr_matrix((w,(i,j))) would SUM them.
    # scipy drops explicit zeros, so every weight gets +eps with eps*n < 1/4:
    # a path's cost is sum(w) + hops*eps and floor() recovers the exact sum.
    key = src * n + dst
    order = np.lexsort((wt, key))
    key_s, wt_s = key[order], wt[order]
    first = np.ones(len(key_s), bool)
    first[1:] = key_s[1:] != key_s[:-1]
    ks, ws = key_s[first], wt_s[first]
    i, j = ks // n, ks % n
    eps = 1.0 / (4.0 * max(n, 1))
    data = ws.astype(np.float64) + eps  # strictly positive; integer part exact
    A = sp.csr_matrix((data, (i, j)), shape=(n, n))
    dist = csgraph.dijkstra(A, directed=True, indices=s)
    sssp = np.where(np.isinf(dist), INF, np.floor(dist)).astype(np.int64)
    B = sp.csr_matrix((np.ones(len(i)), (i, j)), shape=(n, n))
    hops = csgraph.shortest_path(B, directed=True, unweighted=True, indices=s)
    bfs = np.where(np.isinf(hops), INF, hops).astype(np.int64)
    ncomp, lab = csgraph.connected_components(B, directed=True, connection="weak")
    minid = np.full(ncomp, n, np.int64)
    np.minimum.at(minid, lab, np.arange(n))
    return sssp, bfs, minid[lab], ncomp
