"""Concurrent calls on one graph (the paper's
asynchronous BFS/SSSP kernels): graph_share views and
falcon_run_many.  Every job of a concurrent batch must equal the oracle
bit-exactly, whatever else runs next to it."""
import threading

import numpy as np
import pytest

import graphgen as gg
import oracle

pytestmark = pytest.mark.gpu

ALL_JOBS = [("sssp", "vertex"), ("sssp", "edge"), ("sssp", "worklist"), ("sssp", "delta"),
            ("bfs", "vertex"), ("bfs", "edge"), ("bfs", "worklist"),
            ("cc", "vertex"), ("cc", "edge"), ("cc", "worklist")]


def _oracle(algo, G, s):
    if algo == "sssp":
        return oracle.sssp(G.row_off, G.col, G.w, s)
    if algo == "bfs":
        return oracle.bfs(G.row_off, G.col, s)
    return oracle.cc(G.row_off, G.col)


def _ragged():
    s, d, w = gg.er_edges(100_003, 400_011, 77)
    return gg.from_edges("ragged", 100_003, s, d, w, seed=77)


GRAPHS = {"tiny": lambda: gg.config("tiny"), "rand-s": lambda: gg.config("rand-s"),
          "rmat-s": lambda: gg.config("rmat-s"), "grid-s": lambda: gg.config("grid-s"), "ragged": _ragged}
_cache = {}


def _graph(name):
    if name not in _cache:
        _cache[name] = GRAPHS[name]()
    return _cache[name]


@pytest.mark.parametrize("name", list(GRAPHS))
def test_run_many_all_jobs(gpu_lib, name):
    """All 10 (algo, style) jobs at once on a graph and 9 views of it."""
    fb = gpu_lib
    G = _graph(name)
    g = fb.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0)
    handles = [g] + [fb.graph_share(g) for _ in range(len(ALL_JOBS) - 1)]
    outs = [np.full(G.n, -7, np.int32) for _ in ALL_JOBS]
    jobs = [(h, a, s, G.source, o) for h, (a, s), o in zip(handles, ALL_JOBS, outs)]
    for rep in range(2):   # cached CUDA graphs of every handle on the second pass
        stats = fb.falcon_run_many(jobs)
        for (a, s), o, st in zip(ALL_JOBS, outs, stats):
            exp = _oracle(a, G, G.source)
            assert np.array_equal(o, exp), f"{name}/{a}/{s} rep{rep}: {np.flatnonzero(o != exp)[:10]}"
            assert st.iterations >= 1 and st.ms > 0
    for h in handles[1:]:
        fb.graph_free(h)
    fb.graph_free(g)


def test_views_from_threads(gpu_lib):
    """Host threads calling the parent and its views at the same time."""
    fb = gpu_lib
    G = _graph("rmat-s")
    g = fb.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0)
    views = [fb.graph_share(g) for _ in range(3)]
    srcs = [int(s) for s in np.random.default_rng(3).integers(0, G.n, 4)]
    jobs = [(g, "sssp", "worklist", srcs[0]), (views[0], "bfs", "vertex", srcs[1]),
            (views[1], "sssp", "edge", srcs[2]), (views[2], "cc", "vertex", srcs[3])]
    outs = [np.empty(G.n, np.int32) for _ in jobs]
    errs = []

    def work(i):
        h, a, s, src = jobs[i]
        try:
            for _ in range(3):
                fb.run(h, a, s, outs[i], src)
                if not np.array_equal(outs[i], _oracle(a, G, src)):
                    errs.append(f"job {i} {a}/{s} mismatch")
        except Exception as e:   # noqa: BLE001 -- reported below
            errs.append(repr(e))

    ths = [threading.Thread(target=work, args=(i,)) for i in range(len(jobs))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errs, errs
    for v in views:
        fb.graph_free(v)
    fb.graph_free(g)


def test_view_lifecycle_and_errors(gpu_lib):
    fb = gpu_lib
    G = _graph("tiny")
    g = fb.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0)
    v = fb.graph_share(g)
    vv = fb.graph_share(v)            # a view of a view shares the root
    with pytest.raises(fb.FalconError) as e:
        fb.graph_free(g)              # views still live
    assert e.value.name == "INVALID_ARG"
    with pytest.raises(fb.FalconError) as e:
        fb.falcon_set_option(v, "block_bytes", 1 << 20)   # the layout is shared
    assert e.value.name == "UNSUPPORTED"
    fb.falcon_set_option(v, "dense_div", 1)               # schedule options are per handle
    out = np.empty(G.n, np.int32)
    with pytest.raises(fb.FalconError) as e:              # one handle, two jobs
        fb.falcon_run_many([(v, "sssp", "vertex", G.source, out), (v, "bfs", "vertex", G.source, out)])
    assert e.value.name == "INVALID_ARG"
    # a failing job (source >= n) is reported; the launched ones still complete
    o1, o2 = np.empty(G.n, np.int32), np.empty(G.n, np.int32)
    with pytest.raises(fb.FalconError) as e:
        fb.falcon_run_many([(g, "bfs", "worklist", G.source, o1), (vv, "sssp", "vertex", G.n + 5, o2)])
    assert e.value.name == "INVALID_ARG"
    assert np.array_equal(o1, oracle.bfs(G.row_off, G.col, G.source))
    fb.run(vv, "cc", "edge", out, 0)
    assert np.array_equal(out, oracle.cc(G.row_off, G.col))
    fb.graph_free(vv)
    fb.graph_free(v)
    fb.graph_free(g)


def test_run_many_overflow_isolated(gpu_lib):
    """An OVERFLOW in one job does not disturb the other jobs of the batch."""
    fb = gpu_lib
    row_off, col, w = gg.csr_from_edges(4, np.array([0, 1, 2], np.uint32), np.array([1, 2, 3], np.uint32),
                                        np.array([1 << 30] * 3, np.int32))
    g = fb.graph_load_csr(4, 3, row_off, col, w, device=0)
    v = fb.graph_share(g)
    a, b = np.empty(4, np.int32), np.empty(4, np.int32)
    with pytest.raises(fb.FalconError) as e:
        fb.falcon_run_many([(g, "sssp", "vertex", 0, a), (v, "bfs", "edge", 0, b)])
    assert e.value.name == "OVERFLOW"
    assert b.tolist() == [0, 1, 2, 3]
    fb.graph_free(v)
    fb.graph_free(g)
