"""Pins for the CPU oracle (-m "not gpu").

The oracle (oracle/) is pinned to things other than itself:
  * hand-checked examples printed in SPEC.md / derived by hand (tests/golden/),
  * brute force on tiny graphs: Bellman-Ford (n-1 rounds), Floyd-Warshall,
    unit-weight Bellman-Ford for BFS, transitive closure for CC,
  * scipy.sparse.csgraph on medium graphs (min-combined duplicates),
  * O(m) certificates (feasibility + tightness, level parents, CC labels),
  * special cases: unit weights => SSSP == BFS, m=0, self loops/duplicates,
    vertex relabelling, overflow.
"""
import numpy as np
import pytest

import graphgen as gg
import oracle
from common import (INF, bellman_ford, cert_bfs, cert_cc, cert_sssp, closure_cc, floyd_warshall_row,
                    golden_files, load_golden, scipy_reference)


# ------------------------------------------------------------------ golden
@pytest.mark.parametrize("fname", golden_files())
def test_golden(fname):
    g = load_golden(fname)
    row_off, col, w = gg.csr_from_edges(g.n, g.src, g.dst, g.w)
    assert g.cite, "golden fixture without citation"
    if "row_off" in g.expect:
        assert np.array_equal(row_off.astype(np.int64), g.expect["row_off"])
    if "sssp" in g.expect:
        assert np.array_equal(oracle.sssp(row_off, col, w, g.source), g.expect["sssp"])
    if "bfs" in g.expect:
        assert np.array_equal(oracle.bfs(row_off, col, g.source), g.expect["bfs"])
    if "cc" in g.expect:
        assert np.array_equal(oracle.cc(row_off, col), g.expect["cc"])
    if "mst" in g.expect:
        tot, ne, lab = oracle.mst(row_off, col, w)
        assert [tot, ne] == g.expect["mst"].tolist()
        assert np.array_equal(lab, oracle.cc(row_off, col))


# ------------------------------------------------------------------ brute force
def _tiny_graphs(count=220, seed=7):
    rng = np.random.default_rng(seed)
    out = []
    for k in range(count):
        n = int(rng.integers(1, 65))
        m = int(rng.integers(0, 4 * n + 1)) if k % 11 else 0
        src = rng.integers(0, n, m).astype(np.uint32)
        dst = rng.integers(0, n, m).astype(np.uint32)
        wmax = [1, 3, 100, 1 << 20][k % 4]
        w = rng.integers(0, wmax + 1, m).astype(np.int32)  # zeros, self loops, duplicates allowed
        s = int(rng.integers(0, n))
        out.append((n, src, dst, w, s))
    return out


@pytest.mark.parametrize("case", range(0, 220, 1))
def test_bruteforce_tiny(case):
    n, src, dst, w, s = _tiny_graphs()[case]
    row_off, col, wc = gg.csr_from_edges(n, src, dst, w)
    d = oracle.sssp(row_off, col, wc, s)
    assert np.array_equal(d, bellman_ford(n, src, dst, w, s))
    assert np.array_equal(d, floyd_warshall_row(n, src, dst, w, s))
    lv = oracle.bfs(row_off, col, s)
    assert np.array_equal(lv, bellman_ford(n, src, dst, np.ones_like(w), s))
    lab = oracle.cc(row_off, col)
    assert np.array_equal(lab, closure_cc(n, src, dst))


def test_bruteforce_c1_tiny_config():
    """C1 (n=1000, m=4000) against Bellman-Ford and the transitive closure."""
    g = gg.config("tiny")
    src, dst, w = g.edges()
    assert np.array_equal(oracle.sssp(g.row_off, g.col, g.w, g.source), bellman_ford(g.n, src, dst, w, g.source))
    assert np.array_equal(oracle.bfs(g.row_off, g.col, g.source),
                          bellman_ford(g.n, src, dst, np.ones_like(w), g.source))
    assert np.array_equal(oracle.cc(g.row_off, g.col), closure_cc(g.n, src, dst))


# ------------------------------------------------------------------ scipy on medium graphs
@pytest.mark.parametrize("name", ["rand-s", "rmat-s", "grid-s"])
def test_scipy_medium(name):
    g = gg.config(name)
    ss, bb, cc, ncomp = scipy_reference(g.row_off, g.col, g.w, g.source)
    d = oracle.sssp(g.row_off, g.col, g.w, g.source)
    lv = oracle.bfs(g.row_off, g.col, g.source)
    lab = oracle.cc(g.row_off, g.col)
    assert np.array_equal(d, ss)
    assert np.array_equal(lv, bb)
    assert np.array_equal(lab, cc)
    cert_sssp(g.row_off, g.col, g.w, g.source, d)
    cert_bfs(g.row_off, g.col, g.source, lv)
    cert_cc(g.row_off, g.col, lab, ncomp)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_scipy_zero_weights_and_duplicates(seed):
    rng = np.random.default_rng(seed)
    n, m = 3000, 12000
    src = rng.integers(0, n, m).astype(np.uint32); dst = rng.integers(0, n, m).astype(np.uint32)
    src = np.concatenate([src, src[:2000]]); dst = np.concatenate([dst, dst[:2000]])  # duplicates
    w = rng.integers(0, 4, len(src)).astype(np.int32)  # many zero weights
    row_off, col, wc = gg.csr_from_edges(n, src, dst, w)
    s = 5
    ss, bb, cc, ncomp = scipy_reference(row_off, col, wc, s)
    d = oracle.sssp(row_off, col, wc, s)
    assert np.array_equal(d, ss)
    assert np.array_equal(oracle.bfs(row_off, col, s), bb)
    assert np.array_equal(oracle.cc(row_off, col), cc)
    cert_sssp(row_off, col, wc, s, d)


# ------------------------------------------------------------------ special cases
def test_unit_weights_sssp_equals_bfs():
    g = gg.config("rmat-s")
    ones = np.ones_like(g.w)
    assert np.array_equal(oracle.sssp(g.row_off, g.col, ones, g.source), oracle.bfs(g.row_off, g.col, g.source))
    assert np.array_equal(oracle.sssp(g.row_off, g.col, None, g.source), oracle.bfs(g.row_off, g.col, g.source))


def test_no_arcs():
    n = 17
    row_off = np.zeros(n + 1, np.uint32); col = np.zeros(0, np.uint32); w = np.zeros(0, np.int32)
    d = oracle.sssp(row_off, col, w, 3)
    exp = np.full(n, INF); exp[3] = 0
    assert np.array_equal(d, exp)
    assert np.array_equal(oracle.bfs(row_off, col, 3), exp)
    assert np.array_equal(oracle.cc(row_off, col), np.arange(n))


def test_self_loops_and_duplicates_change_nothing():
    g = gg.config("rand-s")
    src, dst, w = g.edges()
    rng = np.random.default_rng(0)
    k = 50_000
    extra_s = rng.integers(0, g.n, k).astype(np.uint32)
    pick = rng.integers(0, g.m, k)
    s2 = np.concatenate([src, extra_s, src[pick]])
    d2 = np.concatenate([dst, extra_s, dst[pick]])
    w2 = np.concatenate([w, rng.integers(0, 100, k).astype(np.int32), w[pick] + 5])
    r2, c2, ww2 = gg.csr_from_edges(g.n, s2, d2, w2)
    assert np.array_equal(oracle.sssp(r2, c2, ww2, g.source), oracle.sssp(g.row_off, g.col, g.w, g.source))
    assert np.array_equal(oracle.bfs(r2, c2, g.source), oracle.bfs(g.row_off, g.col, g.source))
    assert np.array_equal(oracle.cc(r2, c2), oracle.cc(g.row_off, g.col))


def test_relabelling_permutes_outputs():
    g = gg.config("grid-s")
    src, dst, w = g.edges()
    rng = np.random.default_rng(3)
    pi = rng.permutation(g.n).astype(np.uint32)
    r2, c2, w2 = gg.csr_from_edges(g.n, pi[src], pi[dst], w)
    d = oracle.sssp(g.row_off, g.col, g.w, g.source)
    d2 = oracle.sssp(r2, c2, w2, int(pi[g.source]))
    assert np.array_equal(d2[pi], d)
    lv = oracle.bfs(g.row_off, g.col, g.source)
    assert np.array_equal(oracle.bfs(r2, c2, int(pi[g.source]))[pi], lv)
    # CC: same partition, labels recomputed as min ids
    lab, lab2 = oracle.cc(g.row_off, g.col), oracle.cc(r2, c2)
    a = lab2[pi]
    # v ~ u in the original iff pi[v] ~ pi[u] in the relabelled graph
    _, inv1 = np.unique(lab, return_inverse=True)
    _, inv2 = np.unique(a, return_inverse=True)
    pairs = set(zip(inv1.tolist(), inv2.tolist()))
    assert len(pairs) == len(set(inv1.tolist())) == len(set(inv2.tolist()))


def test_overflow_detected():
    # path of 3 arcs with weight 2^30 each: distance 3*2^30 >= INF
    n = 4
    row_off, col, w = gg.csr_from_edges(n, np.array([0, 1, 2], np.uint32), np.array([1, 2, 3], np.uint32),
                                        np.array([1 << 30] * 3, np.int32))
    with pytest.raises(oracle.OracleError):
        oracle.sssp(row_off, col, w, 0)


def test_negative_weight_rejected():
    row_off, col, w = gg.csr_from_edges(2, np.array([0], np.uint32), np.array([1], np.uint32),
                                        np.array([-1], np.int32))
    with pytest.raises(oracle.OracleError):
        oracle.sssp(row_off, col, w, 0)


def test_c1_certificates():
    g = gg.config("tiny")
    d = oracle.sssp(g.row_off, g.col, g.w, g.source)
    cert_sssp(g.row_off, g.col, g.w, g.source, d)
    cert_bfs(g.row_off, g.col, g.source, oracle.bfs(g.row_off, g.col, g.source))
    _, _, _, ncomp = scipy_reference(g.row_off, g.col, g.w, g.source)
    cert_cc(g.row_off, g.col, oracle.cc(g.row_off, g.col), ncomp)


def test_certificates_reject_plausible_mistakes():
    """The certificates themselves must catch a dropped term / wrong index."""
    g = gg.config("tiny")
    d = oracle.sssp(g.row_off, g.col, g.w, g.source).astype(np.int64)
    bad = d.copy(); fin = np.flatnonzero((bad != INF) & (np.arange(g.n) != g.source)); bad[fin[0]] += 1
    with pytest.raises(AssertionError):
        cert_sssp(g.row_off, g.col, g.w, g.source, bad)
    bad = d.copy(); bad[fin[1]] -= 1
    with pytest.raises(AssertionError):
        cert_sssp(g.row_off, g.col, g.w, g.source, bad)
    lab = oracle.cc(g.row_off, g.col).astype(np.int64)
    _, _, _, ncomp = scipy_reference(g.row_off, g.col, g.w, g.source)
    bad = lab.copy(); bad[bad == bad.max()] = 0 if bad.max() != 0 else 1
    if not np.array_equal(bad, lab):
        with pytest.raises(AssertionError):
            cert_cc(g.row_off, g.col, bad, ncomp)


# ------------------------------------------------------------------ MST
def _msf_brute(n, src, dst, w):
    """Minimum spanning forest weight by exhaustive search over arc subsets
    (tiny graphs only): the lightest acyclic subset with n - #components arcs."""
    import itertools
    src = [int(x) for x in src]; dst = [int(x) for x in dst]; w = [int(x) for x in w]
    comps = len(set(closure_cc(n, src, dst).tolist())) if n else 0
    k = n - comps
    best = None
    for sub in itertools.combinations(range(len(src)), k):
        par = list(range(n))

        def f(x):
            while par[x] != x:
                x = par[x]
            return x
        ok = True
        for e in sub:
            a, b = f(src[e]), f(dst[e])
            if a == b:
                ok = False
                break
            par[a] = b
        if ok:
            tot = sum(w[e] for e in sub)
            best = tot if best is None or tot < best else best
    return (best if best is not None else 0), k


def _msf_prim(n, src, dst, w):
    """Prim's algorithm (dense O(n^2)) per component on the symmetrised,
    min-combined adjacency -- a different textbook algorithm than Kruskal."""
    big = np.iinfo(np.int64).max
    A = np.full((n, n), big, dtype=np.int64)
    for u, v, x in zip(np.asarray(src, np.int64), np.asarray(dst, np.int64), np.asarray(w, np.int64)):
        if u != v and x < A[u, v]:
            A[u, v] = A[v, u] = x
    done = np.zeros(n, bool)
    tot = edges = 0
    for r in range(n):
        if done[r]:
            continue
        key = A[r].copy()
        done[r] = True
        while True:
            cand = np.where(~done & (key < big))[0]
            if len(cand) == 0:
                break
            v = cand[np.argmin(key[cand])]
            tot += int(key[v]); edges += 1
            done[v] = True
            key = np.minimum(key, A[v])
    return tot, edges


@pytest.mark.parametrize("case", range(0, 220, 1))
def test_mst_tiny_prim_and_brute(case):
    n, src, dst, w, _ = _tiny_graphs()[case]
    row_off, col, wc = gg.csr_from_edges(n, src, dst, w)
    tot, ne, lab = oracle.mst(row_off, col, wc)
    assert (tot, ne) == _msf_prim(n, src, dst, w)
    assert np.array_equal(lab, oracle.cc(row_off, col))
    if len(src) <= 12 and n <= 9:
        assert (tot, ne) == _msf_brute(n, src, dst, w)


def test_mst_brute_many_tiny():
    rng = np.random.default_rng(470)
    for _ in range(300):
        n = int(rng.integers(1, 8)); m = int(rng.integers(0, 11))
        src = rng.integers(0, n, m).astype(np.uint32); dst = rng.integers(0, n, m).astype(np.uint32)
        w = rng.integers(0, 5, m).astype(np.int32)   # many ties and zeros
        row_off, col, wc = gg.csr_from_edges(n, src, dst, w)
        tot, ne, _ = oracle.mst(row_off, col, wc)
        assert (tot, ne) == _msf_brute(n, src, dst, w)


@pytest.mark.parametrize("name", ["rand-s", "rmat-s", "grid-s"])
def test_mst_scipy_medium(name):
    """scipy.sparse.csgraph.minimum_spanning_tree on the symmetrised graph with
    min-combined duplicates (weights >= 1 here: scipy drops zero entries)."""
    import scipy.sparse as sp
    from scipy.sparse.csgraph import minimum_spanning_tree
    G = gg.config(name)
    src = np.repeat(np.arange(G.n), np.diff(G.row_off.astype(np.int64)))
    dst = G.col.astype(np.int64); w = G.w.astype(np.int64)
    keep = src != dst
    a = np.minimum(src, dst)[keep]; b = np.maximum(src, dst)[keep]; w = w[keep]
    key = a * G.n + b
    order = np.lexsort((w, key))
    key, w = key[order], w[order]
    first = np.r_[True, key[1:] != key[:-1]]
    key, w = key[first], w[first]          # min weight per undirected pair
    M = sp.csr_matrix((w.astype(np.float64), (key // G.n, key % G.n)), shape=(G.n, G.n))
    T = minimum_spanning_tree(M)
    tot, ne, lab = oracle.mst(G.row_off, G.col, G.w)
    assert tot == int(round(T.sum())) and ne == T.nnz
    assert np.array_equal(lab, oracle.cc(G.row_off, G.col))


def test_mst_unit_weights_and_special_cases():
    G = gg.config("rmat-s")
    tot, ne, lab = oracle.mst(G.row_off, G.col, None)   # all weights 1
    comps = len(np.unique(oracle.cc(G.row_off, G.col)))
    assert tot == ne == G.n - comps
    ro = np.zeros(6, np.uint32)                          # no arcs: every vertex its own tree
    assert oracle.mst(ro, np.zeros(0, np.uint32), np.zeros(0, np.int32))[:2] == (0, 0)
    with pytest.raises(oracle.OracleError):
        oracle.mst(np.array([0, 1], np.uint32), np.array([0], np.uint32), np.array([-1], np.int32))
