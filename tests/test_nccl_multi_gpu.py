"""The partitioned path over REAL NCCL ranks, one process per GPU (SURVEY.md
§8(e)): bench.py --mode partition under torchrun with 2 ranks, every rank
loading only its row slice (FALCON_LOAD_SLICE) and returning its owned slice;
the concatenated slices must equal the oracle bit-exactly.  Skipped on boxes
with fewer than two GPUs (this build's GPU boxes have one: the per-rank path
is covered there by loopback ranks, tests/test_loopback_gpu.py)."""
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


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("cfg", ["rand-s", "rmat-s", "grid-s"])
def test_partition_two_nccl_ranks(gpu_lib, tmp_path, cfg):
    dump = str(tmp_path / cfg)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "1", "--warmup", "1", "--config", cfg, "--mode", "partition",
           "--no-e2e", "--no-cpu-baseline", "--dump", dump]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    G = gg.config(cfg)
    meta = json.load(open(os.path.join(dump, "meta.json")))
    for a, s in meta["runs"]:
        exp = oracle.run(a, G)
        got = np.full(G.n, -7, np.int32)
        for rk in range(2):
            rng = json.load(open(os.path.join(dump, f"rank{rk}_range.json")))
            part = np.load(os.path.join(dump, f"rank{rk}_{a}_{s}.npy"))
            got[rng["lo"]:rng["hi"]] = part[:rng["hi"] - rng["lo"]]
        assert np.array_equal(got, exp), (cfg, a, s, np.flatnonzero(got != exp)[:10])
