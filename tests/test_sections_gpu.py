"""The paper's own multi-GPU shapes (PAPER.md:1183-1186,
1587-1597 §3.4 "parallel sections"): different graphs or different
algorithms processed simultaneously, time = the slowest.

* bench.py --mode sections / replica with 2 ranks (gloo process group; the
  ranks share this box's one GPU): every rank's outputs are checked against
  the oracle.
* Two different graphs at once on one GPU (falcon_run_many over two graph
  handles): the pair shape of the paper's Tables tab:multigpucc /
  tab:multigpubfs."""
import glob
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import graphgen as gg
import oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("mode", ["sections", "replica"])
def test_bench_two_ranks_outputs(gpu_lib, tmp_path, mode):
    dump = str(tmp_path / mode)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "1", "--warmup", "1", "--config", "rand-s", "--mode", mode,
           "--dist-backend", "gloo", "--no-e2e", "--no-cpu-baseline", "--dump", dump]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2
    meta = json.load(open(os.path.join(dump, "meta.json")))
    G = gg.config("rand-s")
    exp = {a: oracle.run(a, G) for a in ("sssp", "bfs", "cc")}
    files = sorted(glob.glob(os.path.join(dump, "rank*_*.npy")))
    runs = {tuple(x) for x in meta["runs"]}
    seen = set()
    for f in files:
        rank, a, s = os.path.basename(f)[:-4].split("_")
        assert np.array_equal(np.load(f), exp[a]), f
        seen.add((a, s))
    assert seen == runs   # sections: the runs are dealt over the ranks; replica: every rank runs all
    if mode == "sections":
        assert len(files) == len(runs)
    else:
        assert len(files) == 2 * len(runs)


def test_two_graphs_at_once(gpu_lib):
    """CC / BFS / SSSP on two DIFFERENT graphs launched together (one GPU):
    results equal the one-at-a-time calls and the oracle."""
    fb = gpu_lib
    A, B = gg.config("rand-s"), gg.config("rmat-s")
    ga = fb.graph_load_csr(A.n, A.m, A.row_off, A.col, A.w, device=0)
    gb = fb.graph_load_csr(B.n, B.m, B.row_off, B.col, B.w, device=0)
    for algo, style in (("cc", "worklist"), ("bfs", "vertex"), ("sssp", "delta")):
        oa = torch.empty(A.n, dtype=torch.int32, device="cuda")
        ob = np.empty(B.n, np.int32)
        fb.falcon_run_many([(ga, algo, style, A.source, oa), (gb, algo, style, B.source, ob)])
        assert np.array_equal(oa.cpu().numpy(), oracle.run(algo, A)), algo
        assert np.array_equal(ob, oracle.run(algo, B)), algo
