"""Per-round floor of the fixpoint loop: a directed path 0 -> 1 -> ... -> k-1
inside an n-vertex graph (the other vertices isolated) takes exactly k rounds
with one active vertex each, so ms / rounds is the fixed cost of a round
(launches, the bitmap scan / clear, the advance) at that n.

python tools/round_floor.py [--n 25000000] [--k 2000]
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_1903_01665_b200 as fb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=25_000_000)
ap.add_argument("--k", type=int, default=2000)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
s = np.arange(a.k - 1, dtype=np.uint32)
G = gg.from_edges("path", a.n, s, s + 1, np.ones(a.k - 1, np.int32), source=0)
g = fb.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0, stream=torch.cuda.current_stream(),
                      flags=fb.LOAD_BUILD_COO)
out = torch.empty(G.n, dtype=torch.int32, device="cuda")
for algo, style in (("bfs", "vertex"), ("bfs", "edge"), ("bfs", "worklist"), ("sssp", "vertex"),
                    ("sssp", "worklist"), ("sssp", "delta")):
    fb.run(g, algo, style, out, 0)
    ms = []
    for _ in range(a.reps):
        st = fb.run(g, algo, style, out, 0)
        ms.append(st.ms)
    m = statistics.median(ms)
    print(f"n={a.n} path k={a.k} {algo:4s} {style:8s} {m:8.3f} ms  rounds {st.iterations:5d}  "
          f"{1e3 * m / st.iterations:6.2f} us/round  launches/round {st.kernel_launches / st.iterations:.2f}",
          flush=True)
fb.graph_free(g)
