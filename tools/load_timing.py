"""Time graph_load_csr (host inputs) and the first call of each (algo, style)
(lazy COO / reverse-CSR builds) on a config."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import graphgen as gg
import paper_1903_01665_b200 as fb
G = gg.config(sys.argv[1] if len(sys.argv) > 1 else "rand-25M")
fb.load()
pin = lambda a: torch.from_numpy(a).pin_memory()
h_ro, h_col, h_w = pin(G.row_off), pin(G.col), pin(G.w)
out = torch.empty(G.n, dtype=torch.int32).pin_memory()
for rep in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    g = fb.graph_load_csr(G.n, G.m, h_ro, h_col, h_w, device=0)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"rep{rep} load {1e3*(t1-t):.1f} ms")
    for a in ("sssp", "bfs", "cc"):
        for s in ("vertex", "edge", "worklist"):
            t = time.perf_counter(); st = fb.run(g, a, s, out, G.source); t1 = time.perf_counter()
            print(f"   first {a}/{s}: wall {1e3*(t1-t):.2f} ms  device {st.ms:.2f} ms")
    t = time.perf_counter(); fb.graph_free(g); torch.cuda.synchronize()
    print(f"   free: {1e3*(time.perf_counter()-t):.1f} ms")
