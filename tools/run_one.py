"""Run one (config, algo, style) through the C ABI a few times (for ncu / quick timing).

python tools/run_one.py --config rand-25M --algo sssp --style worklist --reps 2 [--check]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import graphgen as gg
import paper_1903_01665_b200 as fb

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="rand-25M")
ap.add_argument("--algo", default="sssp")
ap.add_argument("--style", default="worklist")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--check", action="store_true", help="compare with the oracle (test infrastructure)")
ap.add_argument("--profile", action="store_true")
ap.add_argument("--delta", type=int, default=0)
a = ap.parse_args()

try:
    from cuda.bindings import runtime as cudart
except Exception:
    from cuda import cudart
for nm in ("cudaDevAttrMaxPersistingL2CacheSize", "cudaDevAttrMaxAccessPolicyWindowSize", "cudaDevAttrL2CacheSize"):
    try:
        print(nm, cudart.cudaDeviceGetAttribute(getattr(cudart.cudaDeviceAttr, nm), 0)[1])
    except Exception as e:
        print(nm, "?", e)
t = time.time()
if a.config.startswith("er:"):   # er:n:m:seed
    _, n_, m_, sd_ = a.config.split(":")
    G = gg.er(int(n_), int(m_), int(sd_))
elif a.config.startswith("rmat:"):
    _, n_, m_, sd_ = a.config.split(":")
    G = gg.rmat(int(n_), int(m_), int(sd_))
else:
    G = gg.config(a.config)
print(f"gen {a.config}: n={G.n} m={G.m} {time.time()-t:.1f}s", flush=True)
g = fb.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0, stream=torch.cuda.current_stream(),
                      flags=fb.LOAD_BUILD_COO)
if a.profile:
    fb.falcon_set_profiling(g, True)
if a.delta:
    fb.falcon_set_delta(g, a.delta)
out = torch.empty(G.n, dtype=torch.int32, device="cuda")
algos = a.algo.split(",")
styles = a.style.split(",")
for algo in algos:
    for style in styles:
        for r in range(a.reps):
            st = fb.run(g, algo, style, out, G.source)
            print(f"{algo}/{style} rep{r}: ms={st.ms:.3f} iters={st.iterations} edges={st.edges_relaxed} "
                  f"upd={st.updates} verts={st.vertices_processed} launches={st.kernel_launches} "
                  f"relax_ms={st.relax_ms:.3f}", flush=True)
        if a.check:
            import oracle
            exp = oracle.run(algo, G)
            assert np.array_equal(out.cpu().numpy(), exp), f"{algo}/{style} mismatch"
            print("  parity ok", flush=True)
