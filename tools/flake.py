"""Flake hunt for falcon_run_many over graph views (tools/calls/r02x.sh).

python tools/flake.py --jobs sssp/vertex,bfs/vertex --iters 300 [--views 1|0] [--config rand-s]
Each iteration loads the graph, makes one view per job (or runs the jobs one
after another on the graph when --views 0), runs the batch twice (the second
time from the cached CUDA graphs) and checks every output against the oracle.
Prints the iteration of the first failure (a CUDA fault ends the process's
context, so one process tests one job set)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import graphgen as gg  # noqa: E402
import oracle  # noqa: E402
import paper_1903_01665_b200 as fb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--jobs", required=True)
ap.add_argument("--iters", type=int, default=300)
ap.add_argument("--views", type=int, default=1, help="1: graph_share views, 2: independent loads, 0: sequential")
ap.add_argument("--config", default="rand-s")
ap.add_argument("--profile", type=int, default=0, help="host-driven rounds (no CUDA graphs / conditional nodes)")
a = ap.parse_args()
G = gg.config(a.config)
jobs = [tuple(j.split("/")) for j in a.jobs.split(",")]
exp = {al: oracle.run(al, G) for al in {j[0] for j in jobs}}
for it in range(a.iters):
    try:
        g = fb.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0)
        if a.views == 2:   # independent loads: no arrays shared between the handles
            hs = [g] + [fb.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0) for _ in range(len(jobs) - 1)]
        else:
            hs = [g] + ([fb.graph_share(g) for _ in range(len(jobs) - 1)] if a.views else [])
        if a.profile:
            for h in hs:
                fb.falcon_set_profiling(h, True)
        outs = [np.full(G.n, -7, np.int32) for _ in jobs]
        for rep in range(2):
            if a.views:
                fb.falcon_run_many([(h, al, st, G.source, o) for h, (al, st), o in zip(hs, jobs, outs)])
            else:
                for (al, st), o in zip(jobs, outs):
                    fb.run(g, al, st, o, G.source)
            for (al, st), o in zip(jobs, outs):
                if not np.array_equal(o, exp[al]):
                    print(f"MISMATCH it={it} rep={rep} {al}/{st}", flush=True)
                    sys.exit(2)
        for h in hs[1:]:
            fb.graph_free(h)
        fb.graph_free(g)
    except Exception as e:   # noqa: BLE001
        print(f"FAIL it={it} jobs={a.jobs} views={a.views}: {e}", flush=True)
        sys.exit(1)
print(f"OK {a.iters} iterations jobs={a.jobs} views={a.views} profile={a.profile}", flush=True)
