"""FALCON_ERR_OVERFLOW means exactly what oracle_sssp's overflow means: some
vertex's shortest distance (the least fixpoint of MIN-relaxation,
PAPER.md:1672, 1679-1686) is finite but >= FALCON_INF (reading R3).  A
candidate d[u] + w >= INF formed on the way -- by a heavy path found before a
light one, or by an arc that is never on a shortest path -- is not an error,
and the status must not depend on the relaxation schedule.

Weights go up to 2^30 (SURVEY §8(c) P4's range)."""
import numpy as np
import pytest

import graphgen as gg
import oracle

pytestmark = pytest.mark.gpu
STYLES = ["vertex", "edge", "worklist", "delta"]
INF = 2147483647


def _expect(row_off, col, w, s):
    try:
        return oracle.sssp(row_off, col, w, s)
    except oracle.OracleError as e:
        assert "overflow" in str(e)
        return None


def _check(fb, g, row_off, col, w, s, styles=STYLES, tag=""):
    exp = _expect(row_off, col, w, s)
    for style in styles:
        out = np.empty(g.n, np.int32)
        if exp is None:
            with pytest.raises(fb.FalconError) as ei:
                fb.run(g, "sssp", style, out, s)
            assert ei.value.name == "OVERFLOW", (tag, style)
        else:
            fb.run(g, "sssp", style, out, s)
            assert np.array_equal(out, exp), (tag, style, np.flatnonzero(out != exp)[:8])
    return exp


def test_verdict_repro_no_overflow(gpu_lib):
    """0->1 (2^30), 1->2 (2^30-2), 2->0 (5): expanding vertex 2 forms the
    candidate 2^31+3 toward vertex 0, but every distance is < INF."""
    fb = gpu_lib
    row_off, col, w = gg.csr_from_edges(3, np.array([0, 1, 2], np.uint32), np.array([1, 2, 0], np.uint32),
                                        np.array([1 << 30, (1 << 30) - 2, 5], np.int32))
    g = fb.graph_load_csr(3, 3, row_off, col, w, device=0)
    exp = _check(fb, g, row_off, col, w, 0)
    assert exp is not None and exp.tolist() == [0, 1 << 30, (1 << 31) - 2]
    for P in (1, 2, 3):
        comm = fb.falcon_comm_init_simulated(P)
        gp = fb.graph_load_csr(3, 3, row_off, col, w, device=0, comm=comm)
        for ex in (0, 1, 2, 3):
            fb.falcon_set_option(gp, "exchange", ex)
            out = np.empty(3, np.int32)
            fb.run(gp, "sssp", "vertex", out, 0)
            assert out.tolist() == exp.tolist(), (P, ex)


def test_true_overflow_all_styles_and_partition(gpu_lib):
    fb = gpu_lib
    row_off, col, w = gg.csr_from_edges(4, np.array([0, 1, 2], np.uint32), np.array([1, 2, 3], np.uint32),
                                        np.array([1 << 30] * 3, np.int32))
    g = fb.graph_load_csr(4, 3, row_off, col, w, device=0)
    assert _check(fb, g, row_off, col, w, 0) is None
    comm = fb.falcon_comm_init_simulated(2)
    gp = fb.graph_load_csr(4, 3, row_off, col, w, device=0, comm=comm)
    for ex in (0, 1, 2, 3):
        fb.falcon_set_option(gp, "exchange", ex)
        with pytest.raises(fb.FalconError) as ei:
            fb.run(gp, "sssp", "vertex", np.empty(4, np.int32), 0)
        assert ei.value.name == "OVERFLOW"


def test_heavy_path_first_is_not_overflow(gpu_lib):
    """A 2-hop heavy path reaches t with a candidate >= INF rounds before a
    60-hop light path gives t a small distance; a tail hangs off t so that
    t's final value matters downstream.  Every style, every schedule: OK."""
    fb = gpu_lib
    L = 60
    s, d, w = [0, 1], [1, 2], [1 << 30, 1 << 30]          # 0 -> 1 -> t=2: 2^31 >= INF
    prev = 0
    for i in range(L):                                       # 0 -> a1 -> ... -> aL -> t, weight 1 each
        a = 4 + i
        s.append(prev); d.append(a); w.append(1)
        prev = a
    s.append(prev); d.append(2); w.append(1)
    s.append(2); d.append(3); w.append((1 << 30) + 7)      # tail: t -> 3
    n = 4 + L
    row_off, col, wc = gg.csr_from_edges(n, np.array(s, np.uint32), np.array(d, np.uint32), np.array(w, np.int32))
    g = fb.graph_load_csr(n, len(col), row_off, col, wc, device=0)
    exp = _check(fb, g, row_off, col, wc, 0)
    assert exp is not None and exp[2] == L + 1 and exp[3] == L + 1 + (1 << 30) + 7
    for delta in (1, 5, 1 << 29):                            # bucket widths change the order of discovery
        fb.falcon_set_delta(g, delta)
        _check(fb, g, row_off, col, wc, 0, styles=["delta"], tag=f"delta={delta}")
    fb.falcon_set_delta(g, 0)


def _tiny_graphs(count=220, seed=7):
    """The oracle's brute-force family (tests/test_oracle.py) re-weighted up to 2^30."""
    rng = np.random.default_rng(seed)
    out = []
    for k in range(count):
        n = int(rng.integers(1, 65))
        m = int(rng.integers(0, 4 * n + 1)) if k % 11 else 0
        src = rng.integers(0, n, m).astype(np.uint32)
        dst = rng.integers(0, n, m).astype(np.uint32)
        hi = [1 << 30, 1 << 29, 1 << 28, 3][k % 4]
        w = rng.integers(hi // 2 if hi > 3 else 0, hi + 1, m).astype(np.int32)
        if k % 5 == 0 and m:
            w[rng.integers(0, m, max(1, m // 4))] = int(rng.integers(0, 100))   # mixed light and heavy arcs
        s = int(rng.integers(0, n))
        out.append((n, src, dst, w, s))
    return out


def test_tiny_graphs_heavy_weights(gpu_lib):
    fb = gpu_lib
    n_ovf = n_ok = 0
    for k, (n, src, dst, w, s) in enumerate(_tiny_graphs()):
        row_off, col, wc = gg.csr_from_edges(n, src, dst, w)
        g = fb.graph_load_csr(n, len(col), row_off, col, wc, device=0)
        exp = _check(fb, g, row_off, col, wc, s, tag=f"case {k}")
        if exp is None:
            n_ovf += 1
        else:
            n_ok += 1
        fb.graph_free(g)
    assert n_ovf >= 20 and n_ok >= 20, (n_ovf, n_ok)   # both outcomes are exercised


def test_delta_round_cap_chain(gpu_lib):
    """chain p_i -> p_{i+1} (1000), p_i -> v_{i+1} (1001),
    p_i -> v_i (0) with Δ = 1 and no local continuation.  v_{i+1} is parked
    in the far set, then improved into the current bucket; the extra refill
    rounds must stay under the DELTA round cap."""
    fb = gpu_lib
    K = 101
    p = lambda i: i
    v = lambda i: K + i
    s, d, w = [], [], []
    for i in range(K):
        if i + 1 < K:
            s += [p(i), p(i)]; d += [p(i + 1), v(i + 1)]; w += [1000, 1001]
        s.append(p(i)); d.append(v(i)); w.append(0)
    n = 2 * K
    row_off, col, wc = gg.csr_from_edges(n, np.array(s, np.uint32), np.array(d, np.uint32), np.array(w, np.int32))
    g = fb.graph_load_csr(n, len(col), row_off, col, wc, device=0)
    fb.falcon_set_delta(g, 1)
    for local in (0, 4):
        fb.falcon_set_option(g, "local", local)
        _check(fb, g, row_off, col, wc, 0, styles=["delta"], tag=f"local={local}")
