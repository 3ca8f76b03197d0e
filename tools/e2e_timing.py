"""Break down one bench.py e2e step (host buffers) with CUDA events and wall
clock: load, each run (incl. lazy layout builds and CUDA-graph capture), free."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_1903_01665_b200 as fb  # noqa: E402

G = gg.config(sys.argv[1] if len(sys.argv) > 1 else "rand-25M")
fb.load()
pin = lambda a: torch.from_numpy(a).pin_memory()
h_ro, h_col, h_w = pin(G.row_off), pin(G.col), pin(G.w)
h_out = torch.empty(G.n, dtype=torch.int32).pin_memory()
stream = torch.cuda.current_stream()
for rep in range(3):
    marks = []
    ev = lambda: (torch.cuda.Event(enable_timing=True), time.perf_counter())

    def mark(name):
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        marks.append((name, e, time.perf_counter()))

    torch.cuda.synchronize()
    mark("start")
    g = fb.graph_load_csr(G.n, G.m, h_ro, h_col, h_w, device=0, stream=stream)
    mark("load")
    for a in ("sssp", "bfs", "cc"):
        for s in ("vertex", "edge", "worklist"):
            fb.run(g, a, s, h_out, G.source)
            mark(f"{a}/{s}")
    fb.graph_free(g)
    mark("free")
    torch.cuda.synchronize()
    tot = marks[0][1].elapsed_time(marks[-1][1])
    print(f"rep{rep}: total device {tot:.1f} ms, wall {1e3 * (marks[-1][2] - marks[0][2]):.1f} ms")
    for (n0, e0, t0), (n1, e1, t1) in zip(marks, marks[1:]):
        print(f"   {n1:14s} device {e0.elapsed_time(e1):7.2f} ms  wall {1e3 * (t1 - t0):7.2f} ms")
