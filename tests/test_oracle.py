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
