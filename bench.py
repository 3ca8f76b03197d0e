#!/usr/bin/env python
"""Benchmark of the fixpoint min-relaxation hot path (SSSP / BFS / CC).

One STEP = one pass of the whole hot path over the workload graph: every
algorithm (SSSP, BFS, CC) in every processing style (VERTEX, EDGE, WORKLIST;
SSSP also DELTA) through the C ABI, i.e. 10 library calls, each doing init ->
device-side fixpoint loop -> output (graph
residency a1 is outside the timed region except in the e2e number).

Metric (BASELINE.json): GTEPS = sum over the step's runs of m_counted / time,
m_counted = arcs whose source is reached (SSSP/BFS; Graph500-style, DESIGN.md
R13) or m (CC).  value is the whole-job aggregate over all ranks.  The line
also carries the roofline of the step's dominant relax kernel and, per graph
class (rand-25M, rmat-10M), the roofline of the best (fastest) style of each
algorithm (`best_style`).

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--config rand-25M]
        python bench.py --impl reference ...   (the CPU oracle, timed on host cores)
Multi-GPU (N>1, torchrun): by default the graph is 1-D vertex-partitioned
over the N GPUs (each rank loads only its row slice, boundary
values travel over NVLink; strong scaling); --mode replica / sections run
the paper's own multi-GPU shapes (independent graphs / "parallel sections",
PAPER.md:1587-1597) instead.  --simulate P runs P partitions on one GPU.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ALGOS = ("sssp", "bfs", "cc")
STYLES = ("vertex", "edge", "worklist", "delta")   # DELTA (Δ-stepping) is SSSP-only
CLASS_CONFIGS = ("rand-25M", "rmat-10M")   # graph classes of the north_star's >= 50 % HBM target (random / RMAT)
HBM_FALLBACK_GBS = 6650.0  # B200_PROFILING.md fallback, used only if MEASURED_PEAKS.json is absent


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="rand-25M")
    ap.add_argument("--algos", default=",".join(ALGOS))
    ap.add_argument("--styles", default=",".join(STYLES))
    ap.add_argument("--impl", default="falcon", choices=["falcon", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-mode", default="many", choices=["many", "calls"],
                    help="e2e step: falcon_run_many over graph views (every job in flight, each result's D2H "
                         "overlapping the other jobs) or one blocking call after another")
    ap.add_argument("--no-classes", action="store_true", help="skip the per-class best-style roofline (rmat-10M)")
    ap.add_argument("--ref-max-steps", type=int, default=3)
    ap.add_argument("--mode", default=None, choices=["replica", "sections", "partition"],
                    help="N>1 (default: partition): partition = one graph 1-D vertex-partitioned over the GPUs, "
                         "each rank loading only its row slice, boundary exchange over NVLink (SURVEY.md §8(e), "
                         "strong scaling); replica = one independent graph per GPU (weak scaling); sections = "
                         "the same graph on every GPU, the step's (algo, style) runs dealt round-robin to the "
                         "GPUs (PAPER.md:1587-1597 'parallel sections', SURVEY §8(f) row 2; time = max over GPUs)")
    ap.add_argument("--simulate", type=int, default=0,
                    help="partition mode on ONE GPU with this many simulated parts (device-side exchange)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for barriers / max-over-ranks (gloo: functional tests of N>1 "
                         "with several ranks sharing one GPU)")
    ap.add_argument("--out", default=None, help="also write the JSON line to this file")
    ap.add_argument("--dump", default=None, help="write every (algo, style) output this rank computed to DIR "
                                                 "(rank<r>_<algo>_<style>.npy; tests compare them with the oracle)")
    return ap.parse_args()


# ------------------------------------------------------------------ helpers
def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


def m_counted(G, algo, out) -> int:
    """Arcs whose source ends with a finite value (SSSP/BFS); m for CC."""
    if algo == "cc":
        return int(G.m)
    deg = np.diff(G.row_off.astype(np.int64))
    return int(deg[np.asarray(out) != 2147483647].sum())


def algorithmic_bytes(algo, style, st, n, m) -> int:
    """Bytes the relax kernels must move for the work they did (SURVEY.md
    §8(d) units): per relaxed arc 12 (SSSP: col, w, gathered
    target value) or 8 (BFS: col, target's visited word); per successful
    update 4 (the atomic write).  Per processed item: VERTEX 8 (row offset,
    own value); queue styles 12 (+ the frontier entry) and 4 per append.
    VERTEX and EDGE read the activity bitmap (n/8 bytes) every round; EDGE
    adds per relaxed arc the 4-byte source id and the 4-byte source value."""
    per_arc = 12 if algo == "sssp" else 8
    V, E, U, R = st["vertices_processed"], st["edges_relaxed"], st["updates"], st["iterations"]
    b = E * per_arc + U * 4
    if style == "vertex":
        b += V * 8 + R * n // 8
    elif style == "edge":
        b += E * 8 + R * n // 8
    else:
        b += V * 12 + U * 4
    return int(b)


def l2_ops(algo, style, st):
    """L2 operations (in random-gather slots) the relax kernels issue for the
    work they did: one gather per relaxed arc, per successful SSSP update one
    RED.MIN (~4 slots) and one activity-bitmap OR (~1.1 slots), per BFS
    discovery two bitmap ORs (profiles/l2_peaks.json)."""
    pk = json.load(open(os.path.join(ROOT, "profiles", "l2_peaks.json")))
    E, U = st["edges_relaxed"], st["updates"]
    if algo == "sssp":
        return E + U * (pk["red_min_cost_in_gathers"] + pk["red_or_bitmap_cost_in_gathers"])
    return E + U * 2 * pk["red_or_bitmap_cost_in_gathers"]


def one_pass_bytes(algo, G) -> int:
    """Work-efficient lower bound (each arc once): SSSP 12m+8n, BFS/CC 8m+8n."""
    return (12 if algo == "sssp" else 8) * G.m + 8 * G.n


def relax_roofline(cfg, algo, style, st, G, hbm, hbm_src, traffic, traffic_src):
    """Roofline of one call's relax kernels: algorithmic bytes (SURVEY §8(d)
    units, algorithmic_bytes) over the summed relax-kernel time measured
    with CUDA events on the library stream (profiling mode); traffic = ncu
    DRAM bytes per relax launch of the same (class, algo, style) call."""
    b = algorithmic_bytes(algo, style, st, G.n, G.m)
    achieved = b / (st["relax_ms"] * 1e-3) / 1e9
    launches = max(1, st["relax_launches"])
    t = traffic.get(f"{cfg}:{algo}/{style}")
    r = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
         "traffic": t["dram_bytes"] / max(1, t["relax_launches"]) if t else None,
         "kernel": f"relax {algo}/{style}", "config": cfg, "peak_source": hbm_src,
         "relax_ms": st["relax_ms"], "relax_launches": st["relax_launches"], "algorithmic_bytes": b,
         "algorithmic_bytes_per_launch": b / launches}
    if t:
        r["dram_over_algorithmic"] = t["dram_over_alg"]
        r["lts_throughput_pct"] = t["lts_throughput_pct_time_weighted"]
        r["traffic_source"] = traffic_src + " (ncu default cache control: L2 flushed before every launch)"
        for k in ("lts_sectors_per_relaxed_arc", "lts_sectors_atom", "lts_sectors_red", "lts_hit_pct_time_weighted"):
            if k in t:
                r[k] = t[k]
        if "warm" in t:   # the same launches with L2 kept across launches (ncu --cache-control none)
            w = t["warm"]
            r["traffic_warm"] = w["dram_bytes"] / max(1, w["relax_launches"])
            r["dram_over_algorithmic_warm"] = w["dram_over_alg"]
    try:   # secondary ceiling: random L2 operations
        pk = json.load(open(os.path.join(ROOT, "profiles", "l2_peaks.json")))
        ops = l2_ops(algo, style, st)
        ach = ops / (st["relax_ms"] * 1e-3) / 1e9
        r["l2_ops"] = {"achieved": ach, "peak": pk["gather_gops_window_le_64MB"], "unit": "G gather-slots/s",
                       "frac": ach / pk["gather_gops_window_le_64MB"], "ops": ops,
                       "peak_source": "profiles/l2_peaks.json (tools/l2probe3.cu)"}
    except (OSError, KeyError, ValueError):
        pass
    return r


def best_block(cfg, G, g, med, prof, fb, hbm, hbm_src, traffic, traffic_src, algos, out):
    """Per algorithm: the fastest style by median ms and the roofline of its
    relax kernels (one profiled call unless the step's profile has it)."""
    blk = {}
    for a in algos:
        cands = {s: ms for (aa, s), ms in med.items() if aa == a}
        if not cands:
            continue
        s = min(cands, key=cands.get)
        st = prof[(a, s)][0] if prof and (a, s) in prof else None
        if st is None:
            fb.falcon_set_profiling(g, True)
            st = fb.run(g, a, s, out, G.source).as_dict()
            fb.falcon_set_profiling(g, False)
        r = relax_roofline(cfg, a, s, st, G, hbm, hbm_src, traffic, traffic_src)
        r.update({"style": s, "ms": cands[s], "ms_by_style": {k: round(v, 4) for k, v in cands.items()},
                  "one_pass_eff": one_pass_bytes(a, G) / (cands[s] * 1e-3) / 1e9 / hbm,
                  "edges_relaxed_over_m": st["edges_relaxed"] / max(1, G.m), "iterations": st["iterations"]})
        blk[a] = r
    return blk


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()   # the timed region starts once the sampler is producing rows
            while not self.rows and time.time() - t0 < 10 and self.proc.poll() is None:
                time.sleep(0.02)
            self.n0 = len(self.rows)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            t0 = time.time()   # at least two samples taken while the timed region ran
            while len(self.rows) < self.n0 + 2 and time.time() - t0 < 2 and self.proc.poll() is None:
                time.sleep(0.02)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, nm in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def traffic_table():
    """ncu DRAM bytes of the relax kernels per (class, algo, style) call
    (tools/traffic.py, committed under profiles/), newest round first."""
    import glob
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")), reverse=True):
        try:
            calls = json.load(open(p))["calls"]
        except (OSError, KeyError, ValueError):
            continue
        # the same calls measured warm (ncu --cache-control none: L2 kept
        # across launches as in a real run), when that table exists
        try:
            warm = json.load(open(p.replace("_traffic.json", "_traffic_warm.json")))["calls"]
            for k, v in calls.items():
                if k in warm:
                    v["warm"] = warm[k]
        except (OSError, KeyError, ValueError):
            pass
        return calls, os.path.relpath(p, ROOT)
    return {}, None


# ------------------------------------------------------------------ CPU oracle legs
def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_pass(G, algos):
    """One oracle pass: each algorithm once, single-threaded, the three
    concurrently in host threads (ctypes releases the GIL).  Each oracle's own
    wall time is taken on its thread with the monotonic (steady) clock.
    Returns (m_counted total, pass wall seconds, threads, per-oracle seconds)."""
    import oracle
    res, per = {}, {}

    def one(a):
        t0 = time.perf_counter()   # CLOCK_MONOTONIC
        res[a] = oracle.run(a, G)
        per[a] = time.perf_counter() - t0

    ths = [threading.Thread(target=one, args=(a,)) for a in algos]
    t0 = time.perf_counter()
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    dt = time.perf_counter() - t0
    return sum(m_counted(G, a, res[a]) for a in algos), dt, len(algos), per


def reference_arm(args, rank, world):
    """--impl reference: the oracle, as it stands, on the host cores."""
    import graphgen as gg
    if rank != 0:
        return
    algos = [a for a in args.algos.split(",") if a]
    G = gg.config(args.config)
    tiny = gg.config("tiny")
    for _ in range(args.warmup):          # warm-up on the tiny config (page-in, caches)
        oracle_pass(tiny, algos)
    steps = max(1, min(args.steps, args.ref_max_steps))
    tot_m, tot_t, cores, per = 0, 0.0, len(algos), {}
    for _ in range(steps):
        mc, dt, cores, per = oracle_pass(G, algos)
        tot_m += mc
        tot_t += dt
    value = tot_m / tot_t / 1e9
    sample = (f"{steps} step(s) of one oracle pass ({'+'.join(algos)}, one algorithm per host thread) over "
              f"{args.config}; warm-up on 'tiny'")
    line = {"impl": "reference", "metric": "SSSP/BFS/CC GTEPS (aggregate over runs per step)", "value": value,
            "unit": "GTEPS", "n_gpus": world, "steps": steps, "steps_requested": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot_t / steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "int32", "data": "synthetic",
            "config": {"workload": args.config, "n": G.n, "m": G.m, "algos": algos, "styles": ["oracle"]},
            "cpu_baseline": {"value": value, "unit": "GTEPS", "cores": cores, "kind": "oracle", "sample": sample,
                             "per_oracle_s": per, "cpu_model": cpu_model(), "host_threads": os.cpu_count()},
            "e2e": {"value": value, "unit": "GTEPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line, args)


def emit(line, args):
    s = json.dumps(line)
    print(s, flush=True)
    if args.out:
        with open(args.out, "w") as f:
            f.write(s + "\n")


# ------------------------------------------------------------------ GPU arm
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference_arm(args, rank, world)

    import torch
    import graphgen as gg
    import paper_1903_01665_b200 as fb

    assert torch.cuda.is_available(), "bench.py needs a CUDA device"
    local = local % torch.cuda.device_count()   # one rank per GPU; ranks may share a GPU in functional tests
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    fb.load()
    algos = [a for a in args.algos.split(",") if a]
    styles = [s for s in args.styles.split(",") if s]

    if args.mode is None:
        args.mode = "partition" if world > 1 else "single"
    partition = args.mode == "partition" or args.simulate > 0
    # Workload: the BASELINE.json config; replica r uses seed + r (weak scaling);
    # partition mode: the same graph on every rank (each keeps its rows).
    sections = args.mode == "sections" and not partition
    if world > 1 and rank > 0 and not partition and not sections:
        base = lambda: gg.config(args.config)
        G = {"rand-25M": lambda: gg.er(25_000_000, 100_000_000, 25 + rank, name="rand-25M"),
             "rmat-10M": lambda: gg.rmat(10_000_000, 100_000_000, 10 + rank, name="rmat-10M"),
             "grid-24M": lambda: gg.grid(6000, 4000, 24 + rank, name="grid-24M")}.get(args.config, base)()
    else:
        G = gg.config(args.config)
    stream = torch.cuda.current_stream()
    comm = None
    if partition:
        if args.simulate > 0:
            comm = fb.falcon_comm_init_simulated(args.simulate)
        else:
            obj = [fb.falcon_comm_unique_id() if rank == 0 else None]
            if dist:
                dist.broadcast_object_list(obj, src=0)
            comm = fb.falcon_comm_init(world, rank, obj[0], local)
        styles = ["vertex"]   # the partitioned path runs the VERTEX round on every part
    if partition and not args.simulate:   # each rank passes only its own rows (FALCON_LOAD_SLICE)
        bounds = fb.falcon_partition(G.row_off, world)
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        base, top = int(G.row_off[lo]), int(G.row_off[hi])
        g = fb.graph_load_csr(hi - lo, top - base, (G.row_off[lo:hi + 1] - base).astype(np.uint32),
                              G.col[base:top], G.w[base:top], device=local, stream=stream, flags=fb.LOAD_SLICE,
                              comm=comm)
    else:
        g = fb.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=local, stream=stream,
                              flags=0 if partition else fb.LOAD_BUILD_COO, comm=comm)
    out = torch.empty(g.out_len, dtype=torch.int32, device="cuda")
    all_runs = [(a, s) for a in algos for s in styles if s != "delta" or a == "sssp"]   # DELTA is SSSP-only
    runs = all_runs[rank::world] if sections else all_runs   # parallel sections: this GPU's share

    def step(collect=None):
        launches = 0
        for a, s in runs:
            st = fb.run(g, a, s, out, G.source)
            launches += st.kernel_launches
            if collect is not None:
                collect.setdefault((a, s), []).append(st.as_dict())
        return launches

    # m_counted per run (outputs are unique fixpoints: style-independent);
    # a rank's output is its owned slice: count its rows, sum over ranks
    mc = {}
    glo, ghi = fb.graph_owned_range(g) if comm is not None else (0, G.n)
    for a in algos:
        fb.run(g, a, styles[0], out, G.source)
        o = out.cpu().numpy()
        if len(o) == G.n:
            mc[a] = m_counted(G, a, o)
        else:
            deg = np.diff(G.row_off[glo:ghi + 1].astype(np.int64))
            c = int(G.row_off[ghi]) - int(G.row_off[glo]) if a == "cc" else int(deg[o != 2147483647].sum())
            if dist:
                t = torch.tensor([c], dtype=torch.int64, device="cuda" if args.dist_backend == "nccl" else "cpu")
                dist.all_reduce(t)
                c = int(t.item())
            mc[a] = c
    units_per_step = sum(mc[a] for a, _ in (all_runs if sections else runs))   # sections: all GPUs' runs

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    per_run = {}
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        launches = 0
        for _ in range(args.steps):
            launches += step(per_run)
        ev1.record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
    ms_total = ev0.elapsed_time(ev1)
    if dist:
        t = torch.tensor([ms_total], device="cuda" if args.dist_backend == "nccl" else "cpu", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    replicas = world if not (partition or sections) else 1   # partition / sections: one job (strong scaling)
    value = replicas * units_per_step * args.steps / (ms_total * 1e-3) / 1e9

    # ---- roofline of the dominant kernel: one profiled step (host-driven loop,
    # CUDA events around every relax launch on the library stream)
    hbm, hbm_src = peaks()
    traffic, traffic_src = traffic_table()
    prof = {}
    roofline = None
    if not partition and runs:
        fb.falcon_set_profiling(g, True)
        step(prof)
        fb.falcon_set_profiling(g, False)
        shares = {k: v[0]["relax_ms"] for k, v in prof.items()}
        dom = max(shares, key=shares.get)
        roofline = relax_roofline(args.config, dom[0], dom[1], prof[dom][0], G, hbm, hbm_src, traffic, traffic_src)
        roofline["share_of_step"] = prof[dom][0]["relax_ms"] / ms_step
    elif partition:   # partitioned: the whole superstep loop (relax + exchange) of the slowest algorithm
        worst = max(per_run, key=lambda k: statistics.median(x["ms"] for x in per_run[k]))
        x = per_run[worst][-1]
        ms = statistics.median(y["ms"] for y in per_run[worst])
        bytes_dom = algorithmic_bytes(worst[0], "vertex", x, G.n, G.m)
        achieved = bytes_dom / (ms * 1e-3) / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm * (world if not args.simulate else 1),
                    "unit": "GB/s", "frac": achieved / (hbm * (world if not args.simulate else 1)), "traffic": None,
                    "kernel": f"partitioned superstep loop {worst[0]} (relax + exchange, all parts)",
                    "peak_source": hbm_src + (" x ranks" if world > 1 else ""), "algorithmic_bytes": bytes_dom}

    # ---- partitioned runs: exchange volume, supersteps, host round trips,
    # and (rank 0, same run) the 1-GPU time of the same calls on the full graph
    part = None
    if partition:
        names = {1: "dense", 2: "sparse", 3: "fused"}
        info = {}
        for a in algos:
            st = fb.run(g, a, "vertex", out, G.source)
            xb = fb.graph_exchange_bytes(g)
            mode_, steps, checks = fb.graph_partition_info(g)
            info[a] = {"ms": st.ms, "exchange": names.get(mode_, mode_), "exchange_bytes_this_rank": xb,
                       "supersteps": steps, "host_round_trips": checks,
                       "nvlink_frac_of_900GBps": (xb / (st.ms * 1e-3) / 900e9) if st.ms > 0 and not args.simulate
                       else None}
        t1 = None
        if rank == 0:
            g1 = fb.graph_load_csr(G.n, G.m, G.row_off, G.col, G.w, device=local, stream=stream)
            o1 = torch.empty(G.n, dtype=torch.int32, device="cuda")
            t1 = {}
            for a in algos:
                fb.run(g1, a, "vertex", o1, G.source)
                t1[a] = statistics.median(fb.run(g1, a, "vertex", o1, G.source).ms for _ in range(3))
            fb.graph_free(g1)
            del o1
        if dist:
            dist.barrier()
        P_ = world if not args.simulate else args.simulate
        tP = {a: statistics.median(x["ms"] for x in per_run[(a, "vertex")]) for a in algos if (a, "vertex") in per_run}
        part = {"parts": P_, "per_algo": info, "t1_ms_same_run": t1, "tP_ms": tP,
                "t1_over_P_tP": {a: t1[a] / (P_ * tP[a]) for a in tP} if t1 and not args.simulate else None,
                "note": "t1 = the same calls (VERTEX style) on the full graph on rank 0's GPU in this run; "
                        "exchange bytes: this rank's sends (fused: 8 B per remote improvement)"}

    if args.dump:   # outputs of this rank's runs, for tests/test_sections_gpu.py
        os.makedirs(args.dump, exist_ok=True)
        for a, s_ in runs:
            fb.run(g, a, s_, out, G.source)
            np.save(os.path.join(args.dump, f"rank{rank}_{a}_{s_}.npy"), out.cpu().numpy())
        if comm is not None:   # this rank's output is its owned slice [lo, hi) (the full array when simulated)
            json.dump({"lo": int(glo), "hi": int(ghi), "len": int(g.out_len)},
                      open(os.path.join(args.dump, f"rank{rank}_range.json"), "w"))
        if rank == 0:
            json.dump({"config": args.config, "mode": args.mode, "world": world, "source": int(G.source),
                       "runs": [list(r) for r in all_runs]}, open(os.path.join(args.dump, "meta.json"), "w"))

    breakdown = {}
    for (a, s), lst in per_run.items():
        ms = statistics.median(x["ms"] for x in lst)
        x = lst[-1]
        p = prof.get((a, s), [x])[0]
        bts = algorithmic_bytes(a, s, x, G.n, G.m)
        breakdown[f"{a}/{s}"] = {"ms": ms, "gteps": mc[a] / (ms * 1e-3) / 1e9, "iterations": x["iterations"],
                                 "edges_relaxed": x["edges_relaxed"], "updates": x["updates"],
                                 "relax_ms": p["relax_ms"], "alg_GBps_relax": bts / (p["relax_ms"] * 1e-3) / 1e9
                                 if p["relax_ms"] and p["relax_ms"] > 0 else None,
                                 "one_pass_eff": one_pass_bytes(a, G) / (ms * 1e-3) / 1e9 / hbm}

    # ---- best processing style per graph class (north_star: >= 50 % of HBM
    # for the best style on random / RMAT graphs at 1 GPU): the fastest style
    # of each algorithm by median ms, and the roofline of ITS relax kernels
    best = None
    if not partition and world == 1 and not args.no_classes:
        best = {}
        for cfg in CLASS_CONFIGS:
            if cfg == args.config:
                med = {k: statistics.median(x["ms"] for x in v) for k, v in per_run.items()}
                best[cfg] = best_block(cfg, G, g, med, prof, fb, hbm, hbm_src, traffic, traffic_src, algos, out)
            else:
                Gc = gg.config(cfg)
                gc = fb.graph_load_csr(Gc.n, Gc.m, Gc.row_off, Gc.col, Gc.w, device=local, stream=stream,
                                       flags=fb.LOAD_BUILD_COO)
                oc = torch.empty(Gc.n, dtype=torch.int32, device="cuda")
                med = {}
                for a, s_ in all_runs:
                    fb.run(gc, a, s_, oc, Gc.source)   # warm-up (lazy layouts, CUDA graphs)
                    med[(a, s_)] = statistics.median(fb.run(gc, a, s_, oc, Gc.source).ms for _ in range(5))
                best[cfg] = best_block(cfg, Gc, gc, med, None, fb, hbm, hbm_src, traffic, traffic_src, algos, oc)
                fb.graph_free(gc)
                del Gc

    # ---- e2e through the C ABI with HOST buffers (H2D + D2H inside the timed region)
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        sliced = partition and not args.simulate   # a rank copies only its own rows (FALCON_LOAD_SLICE)
        if sliced:
            h_ro = pin((G.row_off[lo:hi + 1] - base).astype(np.uint32))
            h_col, h_w = pin(G.col[base:top]), pin(G.w[base:top])
            e_n, e_m, e_flags = hi - lo, top - base, fb.LOAD_SLICE
        else:
            h_ro, h_col, h_w = pin(G.row_off), pin(G.col), pin(G.w)
            e_n, e_m, e_flags = G.n, G.m, 0
        many = args.e2e_mode == "many" and not partition   # (partitioned graphs have no views)
        h_outs = [torch.empty(g.out_len, dtype=torch.int32).pin_memory() for _ in (runs if many else runs[:1])]
        e_steps = max(1, min(args.steps, 3))

        def e2e_step():
            gh = fb.graph_load_csr(e_n, e_m, h_ro, h_col, h_w, device=local, stream=stream, comm=comm, flags=e_flags)
            if many:
                # the public concurrent-call API: one view per job,
                # every job launched before any is waited on, results copied to pinned
                # host buffers on the views' own streams
                hs = [gh] + [fb.graph_share(gh) for _ in runs[1:]]
                fb.falcon_run_many([(h, a, s, G.source, o) for h, (a, s), o in zip(hs, runs, h_outs)])
                for h in hs[1:]:
                    fb.graph_free(h)
            else:
                for a, s in runs:
                    fb.run(gh, a, s, h_outs[0], G.source)
            fb.graph_free(gh)

        e2e_step()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e_steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        if dist:
            t = torch.tensor([ems], device="cuda" if args.dist_backend == "nccl" else "cpu", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": replicas * units_per_step * e_steps / (ems * 1e-3) / 1e9, "unit": "GTEPS",
               "h2d_bytes_per_step": 4 * (e_n + 1) + 8 * e_m, "d2h_bytes_per_step": 4 * g.out_len * len(runs),
               "steps": e_steps, "ms_per_step": ems / e_steps,
               "mode": "falcon_run_many over graph views" if many else "one falcon_* call after another"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        tot, dt, cores, per = oracle_pass(G, algos)
        cpu = {"value": tot / dt / 1e9, "unit": "GTEPS", "cores": cores, "kind": "oracle",
               "sample": f"one oracle pass ({'+'.join(algos)}, one algorithm per host thread, single-threaded "
                         f"each) over {args.config}: {dt:.1f} s wall",
               "per_oracle_s": {a: round(v, 3) for a, v in per.items()}, "cpu_model": cpu_model(),
               "host_threads": os.cpu_count()}

    if rank == 0:
        line = {"metric": "SSSP/BFS/CC GTEPS (aggregate over runs per step)", "value": value, "unit": "GTEPS",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": "strong" if (partition or sections) else "weak",
                "vs_baseline": None,
                "dtype": "int32", "data": "synthetic",
                "config": {"workload": args.config, "n": G.n, "m": G.m, "source": G.source, "algos": algos,
                           "styles": styles, "runs_per_step": len(all_runs),
                           "parallelism": (f"partition{world}" + (f" (simulated {args.simulate} parts on 1 GPU)"
                                                                   if args.simulate else "")) if partition
                           else (f"sections{world}" if sections and world > 1
                                 else ("replicas" if world > 1 else "single")),
                           "l2": "inputs larger than L2 (CSR+COO %.2f GB vs 126 MB L2); each run re-initialises "
                                 "its value array" % ((4 * (G.n + 1) + 12 * G.m) / 1e9)},
                "roofline": roofline, "best_style": best, "partition": part, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clk.summary(), "per_run": breakdown}
        emit(line, args)
    fb.graph_free(g)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
