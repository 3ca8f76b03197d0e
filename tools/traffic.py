"""DRAM traffic vs algorithmic bytes of the relax kernels, per (class, algo,
style) call -- the `traffic` / DRAM-over-algorithmic figures of bench.py's
roofline blocks.

  1. on the GPU box, under ncu (one GPU):
       ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,\
lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,\
lts__t_sectors_op_read.sum,lts__t_sector_hit_rate.pct --clock-control none --csv --log-file gpurun_out/traffic.csv \
           python tools/traffic.py run --out gpurun_out/traffic_stats.json
     (one call per (class, algo, style) in profiling mode; every call ends
     with exactly one k_finish launch, which delimits the calls in the list)
  2. anywhere:  python tools/traffic.py combine gpurun_out/traffic.csv gpurun_out/traffic_stats.json \
                    > profiles/r02_traffic.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

RELAX = ("k_expand_warp", "k_edge", "k_pull", "k_cc_vertex", "k_cc_edge", "k_cc_rest", "k_persist")
CLASSES = ("rand-25M", "rmat-10M")
RUNS = [("sssp", s) for s in ("vertex", "edge", "worklist", "delta")] + \
       [(a, s) for a in ("bfs", "cc") for s in ("vertex", "edge", "worklist")]


def run(out):
    import torch
    import graphgen as gg
    import paper_1903_01665_b200 as fb
    import bench
    res = []
    for cfg in CLASSES:
        G = gg.config(cfg)
        g = fb.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=0, stream=torch.cuda.current_stream(),
                              flags=fb.LOAD_BUILD_COO)
        o = torch.empty(G.n, dtype=torch.int32, device="cuda")
        fb.falcon_set_profiling(g, True)
        for a, s in RUNS:
            st = fb.run(g, a, s, o, G.source).as_dict()
            st["alg_bytes"] = bench.algorithmic_bytes(a, s, st, G.n, G.m)
            res.append({"class": cfg, "algo": a, "style": s, "stats": st})
        fb.graph_free(g)
        del G
    json.dump(res, open(out, "w"), indent=1)


def combine(csv_path, stats_path):
    import launches
    names, L = launches.load(csv_path)
    stats = json.load(open(stats_path))
    calls, cur = [], []
    for k in sorted(L):
        nm = names[k].split("(")[0].replace("void ", "").replace("fk::", "").strip()
        if nm.startswith("k_finish"):
            calls.append(cur)
            cur = []
        elif nm.startswith(RELAX):
            cur.append((nm, L[k]))
    assert len(calls) == len(stats), (len(calls), len(stats))
    out = {}
    for c, s in zip(calls, stats):
        dram = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for _, d in c)
        t_us = sum(d.get("gpu__time_duration.sum", 0) for _, d in c)
        sect = sum(d.get("lts__t_sectors.sum", 0) for _, d in c)
        atom = sum(d.get("lts__t_sectors_op_atom.sum", 0) for _, d in c)
        red = sum(d.get("lts__t_sectors_op_red.sum", 0) for _, d in c)
        rd = sum(d.get("lts__t_sectors_op_read.sum", 0) for _, d in c)
        hit = [d.get("lts__t_sector_hit_rate.pct", 0) for _, d in c]
        lts = [d.get("lts__throughput.avg.pct_of_peak_sustained_elapsed", 0) for _, d in c]
        wts = [d.get("gpu__time_duration.sum", 0) for _, d in c]
        key = f"{s['class']}:{s['algo']}/{s['style']}"
        out[key] = {"relax_launches": len(c), "dram_bytes": dram, "alg_bytes": s["stats"]["alg_bytes"],
                    "dram_over_alg": dram / max(1, s["stats"]["alg_bytes"]), "lts_sectors": sect,
                    "ncu_relax_us": t_us,
                    "lts_throughput_pct_time_weighted": sum(a * b for a, b in zip(lts, wts)) / max(1e-9, sum(wts)),
                    "lts_throughput_pct_max": max(lts) if lts else 0.0,
                    "lts_sectors_read": rd, "lts_sectors_atom": atom, "lts_sectors_red": red,
                    "lts_hit_pct_time_weighted": sum(a * b for a, b in zip(hit, wts)) / max(1e-9, sum(wts)),
                    "edges_relaxed": s["stats"]["edges_relaxed"], "updates": s["stats"]["updates"],
                    "lts_sectors_per_relaxed_arc": sect / max(1, s["stats"]["edges_relaxed"]),
                    "kernels": sorted({nm.split("(")[0] for nm, _ in c})}
    print(json.dumps({"source": "ncu --metrics (cold-cache, serialised; one call per key in profiling mode): "
                                "tools/traffic.py", "calls": out}, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[sys.argv.index("--out") + 1])
    else:
        combine(sys.argv[2], sys.argv[3])
