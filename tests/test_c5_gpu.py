"""BASELINE.json configs[4] (C5): rand-125M and rmat-50M, 500M arcs each --
the largest inputs -- at one GPU and through the partitioned path (8
simulated parts on the one device, the same partition / relax / exchange /
termination code as 8 NCCL ranks).  Every output equals the oracle bit for
bit (the three oracle algorithms run in parallel host threads)."""
import threading

import numpy as np
import pytest

import graphgen as gg
import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
STYLES = ["vertex", "edge", "worklist"]
_cache = {}


def _config_and_oracle(name):
    if name not in _cache:
        G = gg.config(name)
        exp = {}

        def one(a):
            exp[a] = oracle.run(a, G)

        ths = [threading.Thread(target=one, args=(a,)) for a in ("sssp", "bfs", "cc")]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        _cache[name] = (G, exp)
    return _cache[name]


@pytest.mark.parametrize("name", ["rand-125M", "rmat-50M"])
def test_c5_one_gpu(gpu_lib, name):
    G, exp = _config_and_oracle(name)
    g = gpu_lib.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0)
    out = np.empty(G.n, np.int32)
    for algo in ("sssp", "bfs", "cc"):
        for style in STYLES + (["delta"] if algo == "sssp" else []):
            gpu_lib.run(g, algo, style, out, G.source)
            assert np.array_equal(out, exp[algo]), f"{name}/{algo}/{style}: {np.flatnonzero(out != exp[algo])[:8]}"
    gpu_lib.graph_free(g)


@pytest.mark.parametrize("name", ["rand-125M", "rmat-50M"])
def test_c5_partitioned_8_simulated(gpu_lib, name):
    G, exp = _config_and_oracle(name)
    comm = gpu_lib.falcon_comm_init_simulated(8)
    g = gpu_lib.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0, comm=comm)
    out = np.empty(G.n, np.int32)
    for exchange in (0, 3):   # dense device reduce; fused peer writes
        gpu_lib.falcon_set_option(g, "exchange", exchange)
        for algo in ("sssp", "bfs", "cc"):
            gpu_lib.run(g, algo, "vertex", out, G.source)
            assert np.array_equal(out, exp[algo]), f"{name}/P=8/x{exchange}/{algo}: {np.flatnonzero(out != exp[algo])[:8]}"
    gpu_lib.graph_free(g)
