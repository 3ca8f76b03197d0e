"""EDGE style on COO arrays whose 128-arc chunks span few or many sources
(k_edge checks a chunk's liveness from its precomputed
source range), and the skip_now schedule of the SSSP expansion styles
(DESIGN.md §5.2).  Neither may change an output (reading
R8): every result stays bit-exact with the oracle on graphs made of narrow
chunks only, wide chunks only, a mix of both, and ragged tails (m % 4 != 0,
m < 128)."""
import numpy as np
import pytest

import graphgen as gg
import oracle

pytestmark = pytest.mark.gpu


def _sparse_rows(n, m, seed):
    """Average out-degree m/n < 2: 128-arc chunks span ~128 n/m sources, so
    at m/n = 0.5 about half of them are wider than 255 vertices."""
    s, d, w = gg.er_edges(n, m, seed)
    return gg.from_edges(f"er-{n}-{m}", n, s, d, w, seed=seed)


def _clustered(seed=11):
    """Dense rows (narrow chunks) next to a long run of empty rows (one
    chunk spanning 200K vertices) and a hub whose chunks span 0."""
    rng = np.random.default_rng(seed)
    n = 300_000
    dense_u = rng.integers(0, 50_000, 200_000)
    far_u = rng.integers(250_000, n, 300)
    hub_u = np.full(5_000, 60_000)
    s = np.concatenate([dense_u, far_u, hub_u]).astype(np.uint32)
    d = rng.integers(0, n, len(s)).astype(np.uint32)
    w = rng.integers(0, 101, len(s)).astype(np.int32)
    return gg.from_edges("clustered", n, s, d, w, source=0)


CASES = {
    "narrow": lambda: _sparse_rows(200_003, 800_001, 3),
    "mixed": lambda: _sparse_rows(400_001, 200_002, 4),
    "wide": lambda: _sparse_rows(1_000_003, 100_003, 5),
    "clustered": _clustered,
    "small-m5": lambda: _sparse_rows(7, 5, 6),
    "small-m127": lambda: _sparse_rows(1_000, 127, 7),
    "small-m131": lambda: _sparse_rows(300, 131, 8),
}


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("algo", ["sssp", "bfs"])
def test_edge_chunk_spans_parity(gpu_lib, case, algo):
    G = CASES[case]()
    # a source that reaches something: the smallest vertex with an out-arc
    src = int(np.flatnonzero(np.diff(G.row_off))[0]) if G.m else 0
    g = gpu_lib.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0)
    try:
        out = np.full(G.n, -7, np.int32)
        gpu_lib.run(g, algo, "edge", out, src)
        exp = oracle.sssp(G.row_off, G.col, G.w, src) if algo == "sssp" else oracle.bfs(G.row_off, G.col, src)
        bad = np.flatnonzero(out != exp)
        assert bad.size == 0, (case, algo, bad[:8], out[bad[:8]], exp[bad[:8]])
    finally:
        gpu_lib.graph_free(g)


@pytest.mark.parametrize("case", ["mixed", "clustered"])
@pytest.mark.parametrize("style", ["vertex", "worklist", "delta"])
def test_skip_now_parity(gpu_lib, case, style):
    """skip_now on / off: an SSSP item already marked for the next round is
    expanded then instead of now -- same least fixpoint either way."""
    import graphgen as gg
    for G in (CASES[case](), gg.config("rmat-s")):
        src = G.source
        exp = oracle.sssp(G.row_off, G.col, G.w, src)
        for v in (0, 1):
            g = gpu_lib.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0)
            try:
                gpu_lib.falcon_set_option(g, "skip_now", v)
                out = np.full(G.n, -7, np.int32)
                gpu_lib.run(g, "sssp", style, out, src)
                assert np.array_equal(out, exp), (case, style, v, np.flatnonzero(out != exp)[:8])
            finally:
                gpu_lib.graph_free(g)
