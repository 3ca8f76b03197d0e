"""The paper's multi-target experiment shape (Tables
tab:multigpucc / tab:multigpubfs): one algorithm on two DIFFERENT graphs.
The paper's single-GPU column processes them one after another (time = sum);
its multi-GPU column runs each graph on its own GPU (time = the larger).

Measured here on one B200, graphs resident, median of reps:
  sequential  -- the two calls one after another (the paper's "GPU" column)
  run_many    -- both calls in flight at once on one GPU (falcon_run_many)
  max(tA, tB) -- each call alone; what `bench.py --mode sections` on two
                 GPUs times (the ranks share nothing), the paper's
                 "multi-GPU" column

python tools/pairs.py [--reps 5]
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

PAIRS = [("cc", "rand-25M", "rand-50M", 1234, 826), ("cc", "rmat-10M", "rmat-20M", 1176, 792),
         ("bfs", "grid-14M", "grid-24M", 12569, 9138)]   # (algo, A, B, paper GPU ms, paper multi-GPU ms)

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--style", default=None, help="style for every call (default: the fastest per graph class)")
a = ap.parse_args()
BEST = {"cc": {"rand": "worklist", "rmat": "worklist", "grid": "worklist"},
        "bfs": {"rand": "vertex", "rmat": "vertex", "grid": "worklist"}}

for algo, na, nb, p_gpu, p_multi in PAIRS:
    t = time.time()
    GA, GB = gg.config(na), gg.config(nb)
    print(f"== {algo} {na} + {nb}  (gen {time.time() - t:.1f}s)", flush=True)
    ga = fb.graph_load_csr(GA.n, GA.m, GA.row_off, GA.col, GA.w, device=0, stream=torch.cuda.current_stream())
    gb = fb.graph_load_csr(GB.n, GB.m, GB.row_off, GB.col, GB.w, device=0, stream=torch.cuda.current_stream())
    sa = a.style or BEST[algo][na.split("-")[0]]
    sb = a.style or BEST[algo][nb.split("-")[0]]
    oa = torch.empty(GA.n, dtype=torch.int32, device="cuda")
    ob = torch.empty(GB.n, dtype=torch.int32, device="cuda")

    def wall(fn):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        return 1e3 * (time.perf_counter() - t0)

    one_a = lambda: fb.run(ga, algo, sa, oa, GA.source)
    one_b = lambda: fb.run(gb, algo, sb, ob, GB.source)
    both = lambda: fb.falcon_run_many([(ga, algo, sa, GA.source, oa), (gb, algo, sb, GB.source, ob)])
    for f in (one_a, one_b, both):
        f()   # CUDA graphs captured, layouts built
    ta = [wall(one_a) for _ in range(a.reps)]
    tb = [wall(one_b) for _ in range(a.reps)]
    tseq = [wall(lambda: (one_a(), one_b())) for _ in range(a.reps)]
    tmany = [wall(both) for _ in range(a.reps)]
    med = statistics.median
    print(f"{algo} {na}({sa}) {med(ta):8.3f} ms  {nb}({sb}) {med(tb):8.3f} ms  |  sequential {med(tseq):8.3f}  "
          f"run_many {med(tmany):8.3f}  max {max(med(ta), med(tb)):8.3f} ms  |  paper K40C: GPU {p_gpu} ms, "
          f"multi-GPU {p_multi} ms (host wall clock incl. launch, graphs resident)", flush=True)
    fb.graph_free(ga)
    fb.graph_free(gb)
    del GA, GB
