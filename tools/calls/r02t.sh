# Session 3: BFS WORKLIST bottom-up rounds -- parity, then a same-box A/B (env FALCON_BFS_WL_PULL)
set -x
mkdir -p gpurun_out/t
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/t/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/t/smoke.log
timeout 900 python -m pytest tests/test_bfs_wl_pull_gpu.py tests/test_parity_gpu.py tests/test_round2_gpu.py tests/test_concurrent_gpu.py -q -m gpu -k "bfs or worklist or pull or run_many or views" > gpurun_out/t/tests.log 2>&1; echo "rc=$?" >> gpurun_out/t/tests.log
for p in 1 2; do
  for v in 0 1; do
    timeout 600 python tools/survey.py --configs rand-25M,rmat-10M,grid-24M,rand-125M,rmat-50M --algos bfs --styles worklist,vertex --reps 5 --env FALCON_BFS_WL_PULL=$v > gpurun_out/t/wlpull_${v}_p$p.log 2>&1
  done
done
