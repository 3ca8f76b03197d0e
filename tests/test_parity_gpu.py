"""Parity of the CUDA path (through the C ABI) with the CPU oracle.

Bit-exact equality on every output (all three outputs are unique integer
fixpoints), for SSSP / BFS / CC x VERTEX / EDGE / WORKLIST, on
the SPEC.md goldens, edge cases, reduced-scale graphs that span many tiles
with ragged tails, and the full BASELINE.json configs (rand-25M, rmat-10M,
grid-24M) in the launch configuration bench.py times.
"""
import numpy as np
import pytest
import torch

import graphgen as gg
import oracle
from common import INF, cert_bfs, cert_sssp, golden_files, load_golden

pytestmark = pytest.mark.gpu
ALGOS = ["sssp", "bfs", "cc"]
STYLES = ["vertex", "edge", "worklist"]


def _load(fb, n, row_off, col, w, device_inputs=False):
    if device_inputs:
        t = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()
        return fb.graph_load_csr(n, len(col), t(row_off), t(col), t(w), device=0)
    return fb.graph_load_csr(n, len(col), row_off, col, w, device=0)


def _run(fb, g, algo, style, source, device_out=False):
    if device_out:
        out = torch.empty(g.n, dtype=torch.int32, device="cuda")
        st = fb.run(g, algo, style, out, source)
        return out.cpu().numpy(), st
    out = np.empty(g.n, np.int32)
    st = fb.run(g, algo, style, out, source)
    return out, st


def _oracle(algo, row_off, col, w, s):
    if algo == "sssp":
        return oracle.sssp(row_off, col, w, s)
    if algo == "bfs":
        return oracle.bfs(row_off, col, s)
    return oracle.cc(row_off, col)


# ------------------------------------------------------------------ goldens
@pytest.mark.parametrize("fname", golden_files())
@pytest.mark.parametrize("style", STYLES)
def test_golden(gpu_lib, fname, style):
    gd = load_golden(fname)
    row_off, col, w = gg.csr_from_edges(gd.n, gd.src, gd.dst, gd.w)
    g = _load(gpu_lib, gd.n, row_off, col, w)
    for algo in ALGOS:
        if algo in gd.expect:
            out, _ = _run(gpu_lib, g, algo, style, gd.source)
            assert np.array_equal(out, gd.expect[algo]), (fname, algo, style, out)


# ------------------------------------------------------------------ reduced scale, many tiles
def _ragged():
    # m % 4 == 3 (EDGE tail), n not a multiple of any tile size
    s, d, w = gg.er_edges(100_003, 400_011, 77)
    return gg.from_edges("ragged", 100_003, s, d, w, seed=77)


GRAPHS = {
    "tiny": lambda: gg.config("tiny"),
    "rand-s": lambda: gg.config("rand-s"),
    "rmat-s": lambda: gg.config("rmat-s"),
    "grid-s": lambda: gg.config("grid-s"),
    "ragged": _ragged,
}
_cache = {}


def _graph(name):
    if name not in _cache:
        _cache[name] = GRAPHS[name]()
    return _cache[name]


@pytest.mark.parametrize("name", list(GRAPHS))
@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("style", STYLES)
def test_parity_small(gpu_lib, name, algo, style):
    G = _graph(name)
    exp = _oracle(algo, G.row_off, G.col, G.w, G.source)
    g = _load(gpu_lib, G.n, G.row_off, G.col, G.w)
    out, st = _run(gpu_lib, g, algo, style, G.source)
    assert np.array_equal(out, exp), f"{name}/{algo}/{style}: {np.flatnonzero(out != exp)[:10]}"
    assert st.iterations >= 1 and st.kernel_launches >= 2


@pytest.mark.parametrize("name", list(GRAPHS))
@pytest.mark.parametrize("delta", [0, 1, 7, 50, 100000])
def test_parity_delta_stepping(gpu_lib, name, delta):
    """FALCON_STYLE_DELTA (near queue + far set) reaches the same fixpoint for
    any bucket width, including Δ=1 (Dijkstra-like) and Δ >> max distance
    (plain worklist)."""
    G = _graph(name)
    exp = oracle.sssp(G.row_off, G.col, G.w, G.source)
    g = _load(gpu_lib, G.n, G.row_off, G.col, G.w)
    gpu_lib.falcon_set_delta(g, delta)
    out, st = _run(gpu_lib, g, "sssp", "delta", G.source)
    assert np.array_equal(out, exp), f"{name}/delta={delta}: {np.flatnonzero(out != exp)[:10]}"


# layouts / schedules: (block_bytes, dense_div, block_div).  Small blocks
# force the destination-blocked SSSP layout on reduced graphs (several blocks,
# a ragged last block); dense_div 1 keeps queue styles sparse except for huge
# frontiers, 10**6 makes every round dense (bitmap-driven), 0 never dense;
# block_div 10**6 walks the blocked layout in every dense round, 0 never.
LAYOUTS = [(4096, 64, 10**6), (100_000, 10**6, 10**6), (4 << 20, 1, 8), (0, 64, 8), (32 * 1000 + 4, 0, 10**6),
           (65536, 10**6, 0), (65536, 64, 8)]


@pytest.mark.parametrize("name", ["rand-s", "rmat-s", "grid-s", "ragged", "tiny"])
@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("algo", ["sssp", "bfs"])
def test_parity_layouts(gpu_lib, name, layout, algo):
    """Every processing style reaches the oracle's fixpoint whatever the
    destination blocking and the dense/sparse round switch."""
    G = _graph(name)
    exp = _oracle(algo, G.row_off, G.col, G.w, G.source)
    g = _load(gpu_lib, G.n, G.row_off, G.col, G.w)
    gpu_lib.falcon_set_option(g, "block_bytes", layout[0])
    gpu_lib.falcon_set_option(g, "dense_div", layout[1])
    gpu_lib.falcon_set_option(g, "block_div", layout[2])
    for style in STYLES + (["delta"] if algo == "sssp" else []):
        out, st = _run(gpu_lib, g, algo, style, G.source)
        assert np.array_equal(out, exp), f"{name}/{algo}/{style}/{layout}: {np.flatnonzero(out != exp)[:10]}"
        out2, _ = _run(gpu_lib, g, algo, style, G.source, device_out=True)   # cached graph, second run
        assert np.array_equal(out2, exp), f"{name}/{algo}/{style}/{layout} (rerun)"


@pytest.mark.parametrize("name", ["rand-s", "rmat-s", "grid-s", "ragged", "tiny"])
@pytest.mark.parametrize("dense_div", [16, 10**6, 1])
@pytest.mark.parametrize("wl_noq", [0, 1])
@pytest.mark.parametrize("persist", [0, 1])
def test_parity_worklist_noq(gpu_lib, name, dense_div, wl_noq, persist):
    """WORKLIST dense rounds without claims / queue (frontier handed on in the
    bitmap, rebuilt as a queue when the next round is sparse) reach the same
    fixpoint, with and without persistent small rounds."""
    G = _graph(name)
    g = _load(gpu_lib, G.n, G.row_off, G.col, G.w)
    gpu_lib.falcon_set_option(g, "dense_div", dense_div)
    gpu_lib.falcon_set_option(g, "wl_noq", wl_noq)
    gpu_lib.falcon_set_option(g, "persist", persist)
    for algo in ("sssp", "bfs"):
        exp = _oracle(algo, G.row_off, G.col, G.w, G.source)
        out, _ = _run(gpu_lib, g, algo, "worklist", G.source)
        assert np.array_equal(out, exp), f"{name}/{algo}/dd={dense_div}/noq={wl_noq}: {np.flatnonzero(out != exp)[:10]}"


@pytest.mark.parametrize("name", ["rand-s", "rmat-s", "grid-s", "ragged", "tiny"])
@pytest.mark.parametrize("dense_div", [16, 10**6, 1])
@pytest.mark.parametrize("dl_noq", [0, 1])
@pytest.mark.parametrize("persist", [0, 1])
def test_parity_delta_noq(gpu_lib, name, dense_div, dl_noq, persist):
    """DELTA dense rounds without claims / queue (near targets marked in the
    bitmap, far ones parked; the next round reads the bitmap, a refill round
    builds a queue again) reach the same fixpoint for any bucket width."""
    G = _graph(name)
    exp = oracle.sssp(G.row_off, G.col, G.w, G.source)
    g = _load(gpu_lib, G.n, G.row_off, G.col, G.w)
    gpu_lib.falcon_set_option(g, "dense_div", dense_div)
    gpu_lib.falcon_set_option(g, "dl_noq", dl_noq)
    gpu_lib.falcon_set_option(g, "persist", persist)
    for delta in (0, 1, 7, 10**5):
        gpu_lib.falcon_set_delta(g, delta)
        for local in (0, 4):
            gpu_lib.falcon_set_option(g, "local", local)
            for split in ((0, 2, 64) if delta == 0 else (0,)):   # bucket splits (auto Δ only)
                gpu_lib.falcon_set_option(g, "split_div", split)
                out, _ = _run(gpu_lib, g, "sssp", "delta", G.source)
                assert np.array_equal(out, exp), f"{name}/dd={dense_div}/noq={dl_noq}/Δ={delta}/local={local}/split={split}"
    gpu_lib.falcon_set_option(g, "split_div", 0)
    exp_bfs = oracle.bfs(G.row_off, G.col, G.source)
    gpu_lib.falcon_set_option(g, "bfs_unit", 1)   # BFS WORKLIST as unit-weight DELTA
    out, _ = _run(gpu_lib, g, "bfs", "worklist", G.source)
    assert np.array_equal(out, exp_bfs)


@pytest.mark.parametrize("name", ["rand-s", "rmat-s", "grid-s", "ragged", "tiny"])
@pytest.mark.parametrize("local", [1, 2, 16, 1000])
@pytest.mark.parametrize("dense_div", [32, 1])
def test_parity_local_continuation(gpu_lib, name, local, dense_div):
    """SSSP queue rounds whose warps expand the targets they improved
    themselves (option `local`) reach the same fixpoint: small
    budgets hand most local items back to the queue (claims), large ones
    overflow the warp's stack (compaction / spill); Δ = 1 and Δ = 7 keep most
    targets outside the bucket."""
    G = _graph(name)
    exp = oracle.sssp(G.row_off, G.col, G.w, G.source)
    g = _load(gpu_lib, G.n, G.row_off, G.col, G.w)
    gpu_lib.falcon_set_option(g, "local", local)
    gpu_lib.falcon_set_option(g, "wl_local", local)
    gpu_lib.falcon_set_option(g, "wl_local_max", 1 << 30)
    gpu_lib.falcon_set_option(g, "dense_div", dense_div)
    for delta in (0, 1, 7):
        gpu_lib.falcon_set_delta(g, delta)
        for style in ("worklist", "delta"):
            for rep in range(2):
                out, st = _run(gpu_lib, g, "sssp", style, G.source, device_out=rep == 1)
                assert np.array_equal(out, exp), f"{name}/{style}/local={local}/Δ={delta}: {np.flatnonzero(out != exp)[:10]}"
    exp_bfs = oracle.bfs(G.row_off, G.col, G.source)
    for bfs_unit in (1, 0, -1):   # BFS WORKLIST as unit-weight Δ-stepping (R19): on, off, auto
        gpu_lib.falcon_set_option(g, "bfs_unit", bfs_unit)
        for rep in range(2):
            out, st = _run(gpu_lib, g, "bfs", "worklist", G.source, device_out=rep == 1)
            assert np.array_equal(out, exp_bfs), f"{name}/bfs/local={local}/unit={bfs_unit}: {np.flatnonzero(out != exp_bfs)[:10]}"
            assert st.iterations >= 1
    for style in ("vertex", "edge"):   # the options leave the other styles alone
        out, _ = _run(gpu_lib, g, "bfs", style, G.source)
        assert np.array_equal(out, exp_bfs)
    out, _ = _run(gpu_lib, g, "cc", "worklist", G.source)
    assert np.array_equal(out, oracle.cc(G.row_off, G.col))
    tot, ne, _ = gpu_lib.falcon_mst(g, "vertex")   # after a unit-weight BFS: real weights again
    assert (tot, ne) == oracle.mst(G.row_off, G.col, G.w)[:2]
    out, _ = _run(gpu_lib, g, "sssp", "vertex", G.source)
    assert np.array_equal(out, exp)


def test_load_flags_eager_layouts(gpu_lib):
    """FALCON_LOAD_BUILD_COO / _REVERSE build the derived layouts at load;
    results are the same as with the lazy builds; unknown flags are rejected."""
    G = _graph("rmat-s")
    g = gpu_lib.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0,
                               flags=gpu_lib.LOAD_BUILD_COO | gpu_lib.LOAD_BUILD_REVERSE)
    for algo in ALGOS:
        exp = _oracle(algo, G.row_off, G.col, G.w, G.source)
        for style in STYLES:
            out, _ = _run(gpu_lib, g, algo, style, G.source)
            assert np.array_equal(out, exp)
    with pytest.raises(gpu_lib.FalconError) as e:
        gpu_lib.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0, flags=0x80)
    assert e.value.name == "UNSUPPORTED"


def test_memory_cache_reuse_and_trim(gpu_lib):
    """graph_free returns device memory to the library's cache; a second graph
    of the same shape reuses it; falcon_trim_memory hands it back."""
    import torch
    G = _graph("rand-s")
    g = _load(gpu_lib, G.n, G.row_off, G.col, G.w)
    out, _ = _run(gpu_lib, g, "sssp", "edge", G.source)
    gpu_lib.graph_free(g)
    free0 = torch.cuda.mem_get_info()[0]
    g = _load(gpu_lib, G.n, G.row_off, G.col, G.w)          # served from the cache
    out2, _ = _run(gpu_lib, g, "sssp", "edge", G.source)
    assert np.array_equal(out, out2)
    assert torch.cuda.mem_get_info()[0] >= free0 - (64 << 20)
    gpu_lib.graph_free(g)
    released = gpu_lib.falcon_trim_memory()
    assert released > 0
    assert gpu_lib.falcon_trim_memory() == 0


def test_set_option_rejects_unknown(gpu_lib):
    G = _graph("tiny")
    g = _load(gpu_lib, G.n, G.row_off, G.col, G.w)
    with pytest.raises(gpu_lib.FalconError):
        gpu_lib.falcon_set_option(g, "no_such_option", 1)
    with pytest.raises(gpu_lib.FalconError):
        gpu_lib.falcon_set_option(g, "dense_div", -1)
    for bad in (-2, 2):
        with pytest.raises(gpu_lib.FalconError):
            gpu_lib.falcon_set_option(g, "bfs_unit", bad)


def test_delta_rejects_bfs_cc_and_negative(gpu_lib):
    G = _graph("tiny")
    g = _load(gpu_lib, G.n, G.row_off, G.col, G.w)
    with pytest.raises(gpu_lib.FalconError):
        gpu_lib.falcon_bfs(g, 0, "delta", np.empty(G.n, np.int32))
    with pytest.raises(gpu_lib.FalconError):
        gpu_lib.falcon_cc(g, "delta", np.empty(G.n, np.int32))
    with pytest.raises(gpu_lib.FalconError):
        gpu_lib.falcon_set_delta(g, -1)


def test_device_inputs_and_outputs(gpu_lib):
    G = _graph("rmat-s")
    g = _load(gpu_lib, G.n, G.row_off, G.col, G.w, device_inputs=True)
    for algo in ALGOS:
        exp = _oracle(algo, G.row_off, G.col, G.w, G.source)
        for style in STYLES:
            out, _ = _run(gpu_lib, g, algo, style, G.source, device_out=True)
            assert np.array_equal(out, exp)


def test_repeat_and_profiling_mode_identical(gpu_lib):
    G = _graph("rand-s")
    g = _load(gpu_lib, G.n, G.row_off, G.col, G.w)
    for algo in ALGOS:
        exp = _oracle(algo, G.row_off, G.col, G.w, G.source)
        for style in STYLES:
            a, s1 = _run(gpu_lib, g, algo, style, G.source)
            b, _ = _run(gpu_lib, g, algo, style, G.source)
            gpu_lib.falcon_set_profiling(g, True)
            c, sp = _run(gpu_lib, g, algo, style, G.source)
            gpu_lib.falcon_set_profiling(g, False)
            assert np.array_equal(a, exp) and np.array_equal(b, exp) and np.array_equal(c, exp)
            assert sp.relax_ms > 0 and 1 <= sp.relax_launches <= sp.iterations
            assert s1.relax_ms == -1.0


def test_many_sources(gpu_lib):
    G = _graph("rmat-s")
    g = _load(gpu_lib, G.n, G.row_off, G.col, G.w)
    rng = np.random.default_rng(5)
    for s in rng.integers(0, G.n, 6):
        s = int(s)
        for algo in ("sssp", "bfs"):
            exp = _oracle(algo, G.row_off, G.col, G.w, s)
            for style in STYLES:
                out, _ = _run(gpu_lib, g, algo, style, s)
                assert np.array_equal(out, exp)


# ------------------------------------------------------------------ edge cases
def test_single_vertex_no_arcs(gpu_lib):
    row_off = np.zeros(2, np.uint32); col = np.zeros(0, np.uint32)
    g = gpu_lib.graph_load_csr(1, 0, row_off, col, None, device=0)
    for style in STYLES:
        for algo in ALGOS:
            out, _ = _run(gpu_lib, g, algo, style, 0)
            assert out.tolist() == [0]


def test_no_arcs(gpu_lib):
    n = 5000
    row_off = np.zeros(n + 1, np.uint32); col = np.zeros(0, np.uint32)
    g = gpu_lib.graph_load_csr(n, 0, row_off, col, np.zeros(0, np.int32), device=0)
    for style in STYLES:
        d, _ = _run(gpu_lib, g, "sssp", style, 17)
        exp = np.full(n, INF, np.int32); exp[17] = 0
        assert np.array_equal(d, exp)
        l, _ = _run(gpu_lib, g, "cc", style, 0)
        assert np.array_equal(l, np.arange(n, dtype=np.int32))


def test_isolated_source(gpu_lib):
    G = _graph("rand-s")
    deg = G.out_degree()
    iso = int(np.flatnonzero(deg == 0)[0])
    g = _load(gpu_lib, G.n, G.row_off, G.col, G.w)
    for style in STYLES:
        d, _ = _run(gpu_lib, g, "sssp", style, iso)
        assert d[iso] == 0 and (np.delete(d, iso) == INF).all()


def test_unit_weights_null_w(gpu_lib):
    G = _graph("grid-s")
    g = gpu_lib.graph_load_csr(G.n, G.m, G.row_off, G.col, None, device=0)
    exp = oracle.bfs(G.row_off, G.col, G.source)
    for style in STYLES:
        d, _ = _run(gpu_lib, g, "sssp", style, G.source)
        assert np.array_equal(d, exp)


def test_zero_weights_self_loops_duplicates(gpu_lib):
    rng = np.random.default_rng(11)
    n, m = 20_000, 90_001
    s = rng.integers(0, n, m).astype(np.uint32); d = rng.integers(0, n, m).astype(np.uint32)
    s[:500] = d[:500]  # self loops
    s = np.concatenate([s, s[:7000]]); d = np.concatenate([d, d[:7000]])
    w = rng.integers(0, 3, len(s)).astype(np.int32)
    row_off, col, wc = gg.csr_from_edges(n, s, d, w)
    g = gpu_lib.graph_load_csr(n, len(col), row_off, col, wc, device=0)
    for algo in ALGOS:
        exp = _oracle(algo, row_off, col, wc, 3)
        for style in STYLES:
            out, _ = _run(gpu_lib, g, algo, style, 3)
            assert np.array_equal(out, exp)


def test_star_hub(gpu_lib):
    """One hub with 200k out-arcs (degree far above a tile) plus in-arcs."""
    n = 200_001
    s = np.concatenate([np.zeros(n - 1, np.uint32), np.arange(1, n, dtype=np.uint32)])
    d = np.concatenate([np.arange(1, n, dtype=np.uint32), np.zeros(n - 1, np.uint32)])
    w = (np.arange(len(s)) % 97 + 1).astype(np.int32)
    row_off, col, wc = gg.csr_from_edges(n, s, d, w)
    g = gpu_lib.graph_load_csr(n, len(col), row_off, col, wc, device=0)
    for algo in ALGOS:
        exp = _oracle(algo, row_off, col, wc, 5)
        for style in STYLES:
            out, _ = _run(gpu_lib, g, algo, style, 5)
            assert np.array_equal(out, exp)


def test_overflow_status(gpu_lib):
    row_off, col, w = gg.csr_from_edges(4, np.array([0, 1, 2], np.uint32), np.array([1, 2, 3], np.uint32),
                                        np.array([1 << 30] * 3, np.int32))
    g = gpu_lib.graph_load_csr(4, 3, row_off, col, w, device=0)
    for style in STYLES:
        with pytest.raises(gpu_lib.FalconError) as ei:
            _run(gpu_lib, g, "sssp", style, 0)
        assert ei.value.name == "OVERFLOW"


def test_load_validation(gpu_lib):
    fb = gpu_lib
    ro = np.array([0, 2, 3, 3], np.uint32)
    with pytest.raises(fb.FalconError) as e:
        fb.graph_load_csr(3, 3, ro, np.array([1, 5, 2], np.uint32), None, device=0)
    assert e.value.name == "OUT_OF_RANGE"
    with pytest.raises(fb.FalconError) as e:
        fb.graph_load_csr(3, 3, ro, np.array([1, 2, 2], np.uint32), np.array([1, -1, 1], np.int32), device=0)
    assert e.value.name == "OUT_OF_RANGE"
    with pytest.raises(fb.FalconError) as e:
        fb.graph_load_csr(3, 3, np.array([0, 3, 2, 3], np.uint32), np.array([1, 2, 2], np.uint32), None, device=0)
    assert e.value.name == "OUT_OF_RANGE"
    g = fb.graph_load_csr(3, 3, ro, np.array([1, 2, 2], np.uint32), None, device=0)
    with pytest.raises(fb.FalconError) as e:
        fb.falcon_sssp(g, 3, "vertex", np.empty(3, np.int32))
    assert e.value.name == "INVALID_ARG"
    with pytest.raises(fb.FalconError) as e:
        fb.falcon_bfs(g, 0, 7, np.empty(3, np.int32))
    assert e.value.name == "INVALID_ARG"


# ------------------------------------------------------------------ full BASELINE.json configs
@pytest.mark.slow
@pytest.mark.parametrize("name", ["rand-25M", "rmat-10M", "grid-24M"])
def test_parity_full_config(gpu_lib, name):
    G = gg.config(name)
    g = gpu_lib.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0)
    out = np.empty(G.n, np.int32)
    for algo in ALGOS:
        exp = _oracle(algo, G.row_off, G.col, G.w, G.source)
        for style in STYLES:
            gpu_lib.run(g, algo, style, out, G.source)
            assert np.array_equal(out, exp), f"{name}/{algo}/{style}"
        if algo == "sssp":
            gpu_lib.run(g, "sssp", "delta", out, G.source)
            assert np.array_equal(out, exp), f"{name}/sssp/delta"
        if algo == "sssp":
            cert_sssp(G.row_off, G.col, G.w, G.source, exp)
        elif algo == "bfs":
            cert_bfs(G.row_off, G.col, G.source, exp)
