"""Write the round's judged evidence under profiles/ from a gpurun_out/ capture:
bench line, launch-list summary (per-kernel share of one bench step), ncu
--set full summary + hottest SASS of the dominant kernel, and
profiles/ncu_traffic.json (dram bytes per launch of the dominant kernel,
averaged over the launches of one bench step, same metrics as --set full).

python tools/make_profiles.py r01 [gpurun_out]
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import launches  # noqa: E402

tag = sys.argv[1]
src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
prof = os.path.join(ROOT, "profiles")
bench = json.load(open(os.path.join(src, "bench.json")))
with open(os.path.join(prof, f"{tag}_bench_line.json"), "w") as f:
    json.dump(bench, f)
    f.write("\n")
kernel = bench["roofline"]["kernel"].split()[-1]   # e.g. sssp/edge
out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launches.py"), os.path.join(src, "launches.csv")],
                     capture_output=True, text=True).stdout
open(os.path.join(prof, f"{tag}_launches_summary.txt"), "w").write(out)
subprocess.run(["cp", os.path.join(src, "launches.csv"), os.path.join(prof, f"{tag}_launches_bench_step.csv")])
# dominant relax kernel's template name in the launch list
algo, style = kernel.split("/")
ai = {"sssp": 0, "bfs": 1, "cc": 2}[algo]
name = {"edge": f"k_edge<{ai}, 256,", "vertex": f"k_expand_warp<{ai}, 0,", "worklist": f"k_expand_warp<{ai}, 2,"}[style]
names, L = launches.load(os.path.join(src, "launches.csv"))
sel = [L[k] for k in L if name in names[k]]
traffic = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in sel) / max(1, len(sel))
tj = os.path.join(prof, "ncu_traffic.json")
d = json.load(open(tj)) if os.path.exists(tj) else {}
d[kernel] = {"dram_bytes_per_launch": traffic, "launches": len(sel), "kernel": name,
             "source": f"profiles/{tag}_launches_bench_step.csv (ncu dram__bytes_read.sum + dram__bytes_write.sum, "
                       f"mean over the {len(sel)} launches of one bench step)"}
json.dump(d, open(tj, "w"), indent=1)
for rep, label in ((os.path.join(src, "hot.ncu-rep"), f"{tag}_ncu_full_{algo}_{style}.txt"),):
    if os.path.exists(rep):
        a = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep], capture_output=True,
                           text=True).stdout
        b = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_hot.py"), rep, "20"], capture_output=True,
                           text=True).stdout
        open(os.path.join(prof, label), "w").write(a + "\n-- hottest SASS (warp-stall samples) --\n" + b)
print("traffic per launch", traffic, "over", len(sel), "launches of", name)
