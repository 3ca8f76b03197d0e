"""Generator checks: determinism, CSR invariants, and shapes pinned to
PAPER.md Table 1 (tests/golden/table1.txt) and SPEC.md's generator examples."""
import os

import numpy as np
import pytest

import graphgen as gg
from common import GOLDEN_DIR


def _table1():
    rows = {}
    for line in open(os.path.join(GOLDEN_DIR, "table1.txt")):
        line = line.split("#", 1)[0].strip()
        if line:
            name, n, m, md = line.split()
            rows[name] = (float(n) * 1e6, float(m) * 1e6, int(md))
    return rows


def test_determinism_and_chunk_independence():
    a = gg.er_edges(100_000, 3_000_000, 9)
    b = gg.er_edges(100_000, 3_000_000, 9)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    c = gg.er_edges(100_000, 3_000_000, 10)
    assert not np.array_equal(a[0], c[0])


def _py_splitmix64(x):
    M = (1 << 64) - 1
    x = (x + 0x9E3779B97F4A7C15) & M
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return x, z ^ (z >> 31)


def _py_xoshiro_first(seed):
    M = (1 << 64) - 1
    x, s = seed, []
    for _ in range(4):
        x, z = _py_splitmix64(x)
        s.append(z)
    rotl = lambda v, k: ((v << k) | (v >> (64 - k))) & M
    return (rotl((s[1] * 5) & M, 7) * 9) & M


def test_prng_frozen():
    """splitmix64-seeded xoshiro256** ('documented and frozen'),
    checked against an independent Python transcription of the published
    algorithms (Vigna/Blackman)."""
    x, z = _py_splitmix64(0)
    assert z == 0xE220A8397B1DCDAF  # published first splitmix64 output for seed 0
    for seed in (0, 1, 42, 0x5EED, 2**63 + 5):
        assert gg._L().gg_xoshiro_first(seed) == _py_xoshiro_first(seed)
    # Lemire bounded draw: top 32 bits times k, high word (no rejection for these)
    for seed, k in ((3, 100), (9, 1000), (11, 7)):
        top = _py_xoshiro_first(seed) >> 32
        if ((top * k) & 0xFFFFFFFF) >= k:
            assert gg._L().gg_uniform_first(seed, k) == (top * k) >> 32


def test_er_properties():
    s, d, w = gg.er_edges(1000, 50_000, 3)
    assert (s != d).all(), "self loops must be resampled"
    assert w.min() >= 1 and w.max() <= 100
    assert s.max() < 1000 and d.max() < 1000


def test_spec_er_example():
    # gen_er(25000,100000,42) -> maxDegree in [10,30]
    g = gg.er(25_000, 100_000, 42)
    assert 10 <= g.out_degree().max() <= 30


def test_spec_rmat_skew_example():
    # gen_rmat(2^15, 2^18, 7, (0.57,0.19,0.19,0.05)) -> maxDeg >= 50*avgDeg
    g = gg.rmat(1 << 15, 1 << 18, 7, abcd=(0.57, 0.19, 0.19, 0.05))
    deg = g.out_degree()
    assert deg.max() >= 50 * deg.mean()


def test_csr_invariants():
    g = gg.config("rmat-s")
    assert g.row_off[0] == 0 and (np.diff(g.row_off.astype(np.int64)) >= 0).all()
    assert g.row_off[-1] == len(g.col) == len(g.w)
    assert g.col.max() < g.n
    # stable: within a row, input order is kept
    s, d, w = gg.rmat_edges(1 << 17, 1_310_720, 50)
    order = np.argsort(s, kind="stable")
    assert np.array_equal(g.col, d[order]) and np.array_equal(g.w, w[order])


def test_grid_shape():
    g = gg.grid(60, 40, 24)
    deg = g.out_degree()
    assert deg.max() <= 4
    src, dst, _ = g.edges()
    diff = np.abs(src.astype(np.int64) - dst.astype(np.int64))
    assert set(np.unique(diff).tolist()) <= {1, 60}
    # symmetric: both arcs with one weight
    fw = set(zip(src.tolist(), dst.tolist(), g.w.tolist()))
    assert all((v, u, x) in fw for (u, v, x) in fw)


def test_pick_source_has_out_arc():
    g = gg.config("rmat-s")
    s = g.source
    assert g.row_off[s + 1] > g.row_off[s]


@pytest.mark.slow
def test_table1_rand25m_and_grid():
    t1 = _table1()
    g = gg.config("rand-25M")
    n, m, md = t1["rand-25M"]
    assert g.n == n and g.m == m
    assert abs(int(g.out_degree().max()) - md) <= 3  # Poisson(4) max over 25M: 17-19
    del g
    g = gg.config("grid-24M")
    n, m, _ = t1["USA-full"]
    assert g.n == n and abs(g.m - m) / m < 0.01


@pytest.mark.slow
def test_table1_rmat10m():
    t1 = _table1()
    g = gg.config("rmat-10M")
    n, m, md = t1["rmat-10M"]
    assert g.n == n and g.m == m
    assert abs(int(g.out_degree().max()) - md) / md < 0.15
