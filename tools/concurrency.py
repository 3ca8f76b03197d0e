"""Sequential calls vs falcon_run_many (graph_share views) for the bench's
9 (algo, style) jobs, and for SSSP + BFS pairs (the paper's async experiment,
PAPER.md:1040-1064): wall ms per batch, median of reps.

python tools/concurrency.py --configs rand-25M,grid-24M --reps 3
"""
import argparse
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_1903_01665_b200 as fb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="rand-25M,grid-24M")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()

SETS = {"9 bench jobs": [(x, y) for x in ("sssp", "bfs", "cc") for y in ("vertex", "edge", "worklist")],
        "sssp+bfs worklist": [("sssp", "worklist"), ("bfs", "worklist")],
        "sssp+bfs+cc vertex": [("sssp", "vertex"), ("bfs", "vertex"), ("cc", "vertex")]}
for cfg in a.configs.split(","):
    G = gg.config(cfg)
    g = fb.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0, flags=fb.LOAD_BUILD_COO)
    views = [fb.graph_share(g) for _ in range(8)]
    hs = [g] + views
    outs = [torch.empty(G.n, dtype=torch.int32, device="cuda") for _ in hs]
    for name, jobs in SETS.items():
        seq, con = [], []
        for r in range(a.reps + 1):
            torch.cuda.synchronize()
            t = time.perf_counter()
            for (al, st), o in zip(jobs, outs):
                fb.run(g, al, st, o, G.source)
            torch.cuda.synchronize()
            seq.append(1e3 * (time.perf_counter() - t))
            t = time.perf_counter()
            fb.falcon_run_many([(h, al, st, G.source, o) for h, (al, st), o in zip(hs, jobs, outs)])
            torch.cuda.synchronize()
            con.append(1e3 * (time.perf_counter() - t))
        s, c = statistics.median(seq[1:]), statistics.median(con[1:])
        print(f"{cfg:9s} {name:20s} sequential {s:9.2f} ms   run_many {c:9.2f} ms   x{s / c:5.2f}", flush=True)
    for v in views:
        fb.graph_free(v)
    fb.graph_free(g)
