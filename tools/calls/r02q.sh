# Session 3: same-box A/B of HEAD (build/head.so: k_pull 12 B spill) vs the working tree (32-bit per-thread
# counters in k_pull, no spill)
set -x
mkdir -p gpurun_out/q2
L=paper_1903_01665_b200/libfalcon.so
cp $L build/wt.so
for p in 1 2; do
  cp build/head.so $L
  timeout 600 python tools/survey.py --configs rand-25M,rmat-10M,rmat-50M --algos bfs --styles vertex --reps 7 > gpurun_out/q2/head_p$p.log 2>&1
  cp build/wt.so $L
  timeout 600 python tools/survey.py --configs rand-25M,rmat-10M,rmat-50M --algos bfs --styles vertex --reps 7 > gpurun_out/q2/wt_p$p.log 2>&1
done
cp build/wt.so $L
timeout 900 python -m pytest tests/test_round2_gpu.py tests/test_parity_gpu.py -q -m gpu -k "bfs or pull or level" > gpurun_out/q2/tests.log 2>&1; echo "rc=$?" >> gpurun_out/q2/tests.log
