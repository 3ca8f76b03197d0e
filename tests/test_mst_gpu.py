"""MST: falcon_mst against the Kruskal oracle --
total weight and forest-edge count bit-exact (both unique for a minimum
spanning forest), min-id tree labels equal to the CC oracle."""
import numpy as np
import pytest

import graphgen as gg
import oracle
from common import golden_files, load_golden

pytestmark = pytest.mark.gpu
STYLES = ["vertex", "edge"]


def _check(fb, g, row_off, col, w, style):
    exp_tot, exp_ne, exp_lab = oracle.mst(row_off, col, w)
    lab = np.full(len(row_off) - 1, -5, np.int32)
    tot, ne, st = fb.falcon_mst(g, style, lab)
    assert (tot, ne) == (exp_tot, exp_ne), (style, tot, ne, exp_tot, exp_ne)
    assert np.array_equal(lab, exp_lab)
    assert st.iterations >= 1
    return st


@pytest.mark.parametrize("fname", [f for f in golden_files() if "mst" in f])
@pytest.mark.parametrize("style", STYLES)
def test_mst_golden(gpu_lib, fname, style):
    gd = load_golden(fname)
    row_off, col, w = gg.csr_from_edges(gd.n, gd.src, gd.dst, gd.w)
    g = gpu_lib.graph_load_csr(gd.n, len(col), row_off, col, w, device=0)
    tot, ne, _ = gpu_lib.falcon_mst(g, style)
    assert [tot, ne] == gd.expect["mst"].tolist()


def _ragged():
    s, d, w = gg.er_edges(100_003, 400_011, 77)
    return gg.from_edges("ragged", 100_003, s, d, w, seed=77)


@pytest.mark.parametrize("name", ["tiny", "rand-s", "rmat-s", "grid-s", "ragged"])
@pytest.mark.parametrize("style", STYLES)
def test_mst_parity(gpu_lib, name, style):
    G = _ragged() if name == "ragged" else gg.config(name)
    g = gpu_lib.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0)
    st = _check(gpu_lib, g, G.row_off, G.col, G.w, style)
    assert st.iterations <= int(np.ceil(np.log2(max(G.n, 2)))) + 2   # Borůvka: components at least halve
    _check(gpu_lib, g, G.row_off, G.col, G.w, style)                 # repeated call


def test_mst_many_tiny(gpu_lib):
    """Random tiny graphs with zero weights, many ties, self loops, duplicates."""
    rng = np.random.default_rng(492)
    for k in range(120):
        n = int(rng.integers(1, 70)); m = int(rng.integers(0, 4 * n + 1)) if k % 9 else 0
        src = rng.integers(0, n, m).astype(np.uint32); dst = rng.integers(0, n, m).astype(np.uint32)
        w = rng.integers(0, [1, 3, 100, 1 << 30][k % 4] + 1, m).astype(np.int32)
        row_off, col, wc = gg.csr_from_edges(n, src, dst, w)
        g = gpu_lib.graph_load_csr(n, len(col), row_off, col, wc, device=0)
        for style in STYLES:
            _check(gpu_lib, g, row_off, col, wc, style)
        gpu_lib.graph_free(g)


def test_mst_unit_weights_and_views(gpu_lib):
    G = gg.config("rmat-s")
    g = gpu_lib.graph_load_csr(G.n, G.m, G.row_off, G.col, None, device=0)
    v = gpu_lib.graph_share(g)
    for h in (g, v):
        tot, ne, _ = gpu_lib.falcon_mst(h, "edge")
        exp = oracle.mst(G.row_off, G.col, None)
        assert (tot, ne) == exp[:2] and tot == ne
    with pytest.raises(gpu_lib.FalconError) as e:
        gpu_lib.falcon_mst(g, "worklist")
    assert e.value.name == "UNSUPPORTED"
    gpu_lib.graph_free(v)
    gpu_lib.graph_free(g)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["rand-25M", "rmat-10M", "grid-24M"])
def test_mst_full_config(gpu_lib, name):
    G = gg.config(name)
    g = gpu_lib.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0)
    exp_tot, exp_ne, exp_lab = oracle.mst(G.row_off, G.col, G.w)
    for style in STYLES:
        lab = np.empty(G.n, np.int32)
        tot, ne, _ = gpu_lib.falcon_mst(g, style, lab)
        assert (tot, ne) == (exp_tot, exp_ne), f"{name}/{style}"
        assert np.array_equal(lab, exp_lab)
