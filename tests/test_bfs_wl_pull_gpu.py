"""BFS WORKLIST with bottom-up rounds (option bfs_wl_pull, DESIGN.md §5.5;
SURVEY §8(a) a5 "optional pull over innbrs when the frontier is large"):
a round may scan the unvisited vertices' in-arcs (`innbrs`)
instead of the queue's out-arcs; the next round reads its items from the
pull round's bitmap.  Levels are the unique hop distances either way
(PAPER.md:1302-1329), so both settings must equal the oracle bit for bit."""
import numpy as np
import pytest

import graphgen as gg
import oracle

pytestmark = pytest.mark.gpu


def _deep(n=1_500, seed=5):
    rng = np.random.default_rng(seed)
    s = list(range(n - 1)) + list(rng.integers(0, n - 2, 3 * n))
    d = list(range(1, n)) + [x + 1 for x in s[n - 1:]]
    nn = n + 37   # unreachable vertices
    return gg.from_edges("deep", nn, np.array(s, np.uint32), np.array(d, np.uint32), None, source=0)


GRAPHS = {"tiny": lambda: gg.config("tiny"), "rand-s": lambda: gg.config("rand-s"),
          "rmat-s": lambda: gg.config("rmat-s"), "grid-s": lambda: gg.config("grid-s"), "deep": _deep}


@pytest.mark.parametrize("name", sorted(GRAPHS))
def test_bfs_worklist_pull_parity(gpu_lib, name):
    G = GRAPHS[name]()
    exp = oracle.bfs(G.row_off, G.col, G.source)
    for v in (1, 0):
        g = gpu_lib.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0)
        try:
            gpu_lib.falcon_set_option(g, "bfs_wl_pull", v)
            for rep in range(2):   # second call: the cached CUDA graph
                out = np.full(G.n, -7, np.int32)
                gpu_lib.run(g, "bfs", "worklist", out, G.source)
                assert np.array_equal(out, exp), (name, v, rep, np.flatnonzero(out != exp)[:8])
        finally:
            gpu_lib.graph_free(g)
