"""Time every (config, algo, style) through the C ABI (median of reps) -- the
performance landscape used to pick what to optimise next.

python tools/survey.py --configs rand-25M,rmat-10M,grid-24M --reps 5 [--env K=V ...]
"""
import argparse
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="rand-25M,rmat-10M,grid-24M")
ap.add_argument("--algos", default="sssp,bfs,cc")
ap.add_argument("--styles", default="vertex,edge,worklist,delta")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--env", nargs="*", default=[])
a = ap.parse_args()
for kv in a.env:
    k, v = kv.split("=", 1)
    os.environ[k] = v

import torch  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_1903_01665_b200 as fb  # noqa: E402

for cfg in a.configs.split(","):
    t = time.time()
    G = gg.config(cfg)
    print(f"== {cfg}: n={G.n} m={G.m} gen {time.time() - t:.1f}s", flush=True)
    g = fb.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0, stream=torch.cuda.current_stream(),
                          flags=fb.LOAD_BUILD_COO)
    out = torch.empty(G.n, dtype=torch.int32, device="cuda")
    for algo in a.algos.split(","):
        for style in a.styles.split(","):
            if style == "delta" and algo != "sssp":
                continue
            if algo == "mst" and style not in ("vertex", "edge"):
                continue
            one = (lambda: fb.falcon_mst(g, style, out)[2]) if algo == "mst" else \
                (lambda: fb.run(g, algo, style, out, G.source))
            one()
            ms = []
            for _ in range(a.reps):
                st = one()
                ms.append(st.ms)
            print(f"{cfg:9s} {algo:4s} {style:8s} med {statistics.median(ms):8.3f} ms  min {min(ms):8.3f}  "
                  f"iters {st.iterations:6d}  edges {st.edges_relaxed / G.m:6.2f} m  upd {st.updates:11d}  "
                  f"launches {st.kernel_launches}", flush=True)
    fb.graph_free(g)
