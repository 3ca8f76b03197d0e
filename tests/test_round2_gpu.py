"""Parity of the round-2 schedule changes with the CPU oracle (bit-exact):
BFS byte levels on both sides of the 255-level switch, the per-round
direction choice and the two pull forms of BFS VERTEX, and CTA-level
expansion of long rows at every threshold.  None of
them may change an output: they only change the order and the placement of
the relaxations (reading R8)."""
import numpy as np
import pytest

import graphgen as gg
import oracle

pytestmark = pytest.mark.gpu

STYLES = ["vertex", "edge", "worklist"]


def _star(n=60_001, seed=3):
    """A hub with n-1 out-arcs, every leaf one arc back and one to the next leaf."""
    leaves = np.arange(1, n, dtype=np.uint32)
    s = np.concatenate([np.zeros(n - 1, np.uint32), leaves, leaves])
    d = np.concatenate([leaves, np.zeros(n - 1, np.uint32), np.where(leaves + 1 < n, leaves + 1, 1).astype(np.uint32)])
    w = (np.arange(len(s)) % 97 + 1).astype(np.int32)
    return gg.from_edges("star", n, s, d, w, source=0)


def _deep(n=1_500, seed=5):
    """A path 0 -> 1 -> ... -> n-1 (level of v = v, so the quads around 255
    mix byte and int32 levels) with extra forward arcs that never shortcut it
    by more than one hop, plus unreachable vertices."""
    rng = np.random.default_rng(seed)
    s = list(range(n - 1))
    d = list(range(1, n))
    extra = rng.integers(0, n - 2, 3 * n)
    s += list(extra)
    d += list(extra + 1)          # parallel copies of path arcs (duplicates)
    back = rng.integers(1, n - 1, n)
    s += list(back)
    d += list(rng.integers(0, back))   # backward arcs (never shorten)
    nn = n + 37                   # 37 isolated, unreachable vertices
    s = np.array(s, np.uint32)
    d = np.array(d, np.uint32)
    w = rng.integers(1, 101, len(s)).astype(np.int32)
    return gg.from_edges("deep", nn, s, d, w, source=0)


GRAPHS = {"tiny": lambda: gg.config("tiny"), "rand-s": lambda: gg.config("rand-s"),
          "rmat-s": lambda: gg.config("rmat-s"), "grid-s": lambda: gg.config("grid-s"),
          "star": _star, "deep": _deep}
_cache = {}


def _graph(name):
    if name not in _cache:
        _cache[name] = GRAPHS[name]()
    return _cache[name]


def _run(fb, g, algo, style, source):
    out = np.full(g.n, -7, np.int32)
    st = fb.run(g, algo, style, out, source)
    return out, st


@pytest.mark.parametrize("style", STYLES)
def test_bfs_levels_across_the_byte_switch(gpu_lib, style):
    """Levels 0..1499 on one graph: below 255 through the byte array, from
    255 on in the int32 array, merged by k_bfs_levels; repeated calls reuse
    the byte array."""
    G = _graph("deep")
    exp = oracle.bfs(G.row_off, G.col, G.source)
    assert exp[:G.n - 37].max() == 1499 and (exp[G.n - 37:] == 2**31 - 1).all()
    g = gpu_lib.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0)
    for rep in range(2):
        out, st = _run(gpu_lib, g, "bfs", style, G.source)
        assert np.array_equal(out, exp), (style, rep, np.flatnonzero(out != exp)[:10])
    # a shallow call after a deep one on the same handle (no stale int32 levels leak in)
    out, _ = _run(gpu_lib, g, "bfs", style, 1200)
    assert np.array_equal(out, oracle.bfs(G.row_off, G.col, 1200))


@pytest.mark.parametrize("name", list(GRAPHS))
@pytest.mark.parametrize("rule,pull_div", [(0, 16), (1, 1), (1, 4), (2, 1), (2, 4), (2, 16), (1, 10**6), (0, 0)])
def test_bfs_vertex_direction_and_pull_forms(gpu_lib, name, rule, pull_div):
    """BFS VERTEX under the cost-model direction (rule 0), and with the pull
    forced whenever the frontier exceeds n / pull_div in the word (1) and the
    compacted (2) pull form -- pull_div 1 pulls every round with a frontier."""
    G = _graph(name)
    exp = oracle.bfs(G.row_off, G.col, G.source)
    g = gpu_lib.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0)
    gpu_lib.falcon_set_option(g, "pull_rule", rule)
    gpu_lib.falcon_set_option(g, "pull_div", pull_div)
    for rep in range(2):
        out, st = _run(gpu_lib, g, "bfs", "vertex", G.source)
        assert np.array_equal(out, exp), (name, rule, pull_div, rep, np.flatnonzero(out != exp)[:10])


@pytest.mark.parametrize("name", ["star", "rmat-s", "rand-s", "grid-s", "tiny"])
@pytest.mark.parametrize("cta_thr", [0, 8, 32, 1024])
def test_cta_level_expansion(gpu_lib, name, cta_thr):
    """Rows longer than cta_thr arcs are expanded by the whole CTA (8 warps);
    cta_thr 8 lists far more long rows than a CTA's 64-entry list holds (the
    rest stay warp-level).  Every style that expands rows, dense and sparse
    rounds (dense_div 10**6 / 0), local-continuation rounds included."""
    G = _graph(name)
    g = gpu_lib.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0)
    gpu_lib.falcon_set_option(g, "cta_thr", cta_thr)
    exp = {"sssp": oracle.sssp(G.row_off, G.col, G.w, G.source), "bfs": oracle.bfs(G.row_off, G.col, G.source)}
    for dense_div in (32, 10**6, 0):
        gpu_lib.falcon_set_option(g, "dense_div", dense_div)
        for algo, styles in (("sssp", ("vertex", "worklist", "delta")), ("bfs", ("vertex", "worklist"))):
            for style in styles:
                out, _ = _run(gpu_lib, g, algo, style, G.source)
                assert np.array_equal(out, exp[algo]), (name, cta_thr, dense_div, algo, style,
                                                         np.flatnonzero(out != exp[algo])[:10])


def test_cta_level_expansion_views_run_many(gpu_lib):
    """Long rows on concurrent views (falcon_run_many), pageable outputs."""
    G = _graph("star")
    g = gpu_lib.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0)
    gpu_lib.falcon_set_option(g, "cta_thr", 16)
    views = [gpu_lib.graph_share(g) for _ in range(3)]
    jobs = [("sssp", "vertex"), ("sssp", "delta"), ("bfs", "vertex"), ("bfs", "worklist")]
    outs = [np.full(G.n, -7, np.int32) for _ in jobs]
    gpu_lib.falcon_run_many([(h, a, s, G.source, o) for h, (a, s), o in zip([g] + views, jobs, outs)])
    for (a, s), o in zip(jobs, outs):
        exp = oracle.sssp(G.row_off, G.col, G.w, G.source) if a == "sssp" else oracle.bfs(G.row_off, G.col, G.source)
        assert np.array_equal(o, exp), (a, s)
    for v in views:
        gpu_lib.graph_free(v)
