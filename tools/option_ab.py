"""A/B one library option on the same graph (same box, one handle per value, interleaved reps).

python tools/option_ab.py --config rmat-10M --algos sssp,bfs --styles vertex,worklist --option cta_thr=0,1024
Configs: the graphgen names, er:n:m:seed, rmat:n:m:seed, star:n (a hub with n-1 out-arcs, every leaf
with one arc back to the hub and one to the next leaf).
"""
import argparse
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_1903_01665_b200 as fb  # noqa: E402


def make(cfg):
    if cfg.startswith("er:"):
        _, n, m, sd = cfg.split(":")
        return gg.er(int(n), int(m), int(sd))
    if cfg.startswith("rmat:"):
        _, n, m, sd = cfg.split(":")
        return gg.rmat(int(n), int(m), int(sd))
    if cfg.startswith("star:"):
        n = int(cfg.split(":")[1])
        leaves = np.arange(1, n, dtype=np.uint32)
        s = np.concatenate([np.zeros(n - 1, np.uint32), leaves, leaves])
        d = np.concatenate([leaves, np.zeros(n - 1, np.uint32), np.where(leaves + 1 < n, leaves + 1, 1).astype(np.uint32)])
        w = (np.arange(len(s)) % 97 + 1).astype(np.int32)
        return gg.from_edges(cfg, n, s, d, w, source=0)
    return gg.config(cfg)


ap = argparse.ArgumentParser()
ap.add_argument("--config", default="rmat-10M")
ap.add_argument("--algos", default="sssp,bfs")
ap.add_argument("--styles", default="vertex,worklist")
ap.add_argument("--option", required=True, help="name=v1,v2,...")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
name, vals = a.option.split("=")
vals = [int(v) for v in vals.split(",")]
t = time.time()
G = make(a.config)
print(f"== {a.config}: n={G.n} m={G.m} gen {time.time() - t:.1f}s  option {name} in {vals}", flush=True)
# one handle per option value (setting an option drops the handle's cached
# CUDA graphs, so switching one handle back and forth would time captures)
hs = {}
for v in vals:
    hs[v] = fb.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0, stream=torch.cuda.current_stream(),
                              flags=fb.LOAD_BUILD_COO)
    fb.falcon_set_option(hs[v], name, v)
out = torch.empty(G.n, dtype=torch.int32, device="cuda")
for algo in a.algos.split(","):
    for style in a.styles.split(","):
        if style == "delta" and algo != "sssp":
            continue
        ms = {v: [] for v in vals}
        work = {}
        ref = None
        for r in range(a.reps + 1):   # rep 0: warm-up (layouts, CUDA graph capture)
            for v in vals:
                st = fb.run(hs[v], algo, style, out, G.source)
                if r:
                    ms[v].append(st.ms)
                    work[v] = (st.iterations, st.edges_relaxed / max(G.m, 1))
                res = out.cpu().numpy().copy()
                if ref is None:
                    ref = res
                assert np.array_equal(res, ref), f"{algo}/{style}: {name}={v} changed the result"
        line = "  ".join(f"{name}={v}: {statistics.median(ms[v]):8.3f} ({work[v][0]} rnd, {work[v][1]:.2f} m)"
                         for v in vals)
        print(f"{a.config:10s} {algo:4s} {style:8s} {line}  ms (median of {a.reps})", flush=True)
for v in vals:
    fb.graph_free(hs[v])
