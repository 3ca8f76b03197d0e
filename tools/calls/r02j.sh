# Session 3: EDGE 8-bit sources (v2) timings + parity, skip_now A/B, run_many stress
set -x
mkdir -p gpurun_out/j
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/j/build.log 2>&1
timeout 300 python tools/survey.py --configs rand-25M,rmat-10M --algos sssp,bfs --styles edge --reps 5 > gpurun_out/j/survey_edge.log 2>&1
timeout 600 python -m pytest tests/test_edge_src8_gpu.py tests/test_parity_gpu.py -q -m gpu -k "edge or src8" > gpurun_out/j/tests_edge.log 2>&1; echo "rc=$?" >> gpurun_out/j/tests_edge.log
for c in rand-25M rmat-10M; do
  timeout 600 python tools/option_ab.py --config $c --algos sssp --styles vertex,worklist,delta --option skip_now=0,1 --reps 5 >> gpurun_out/j/ab_skip_now.log 2>&1
done
for i in 1 2 3 4 5 6 7 8; do
  timeout 600 python -m pytest tests/test_concurrent_gpu.py -x -q > gpurun_out/j/stress_$i.log 2>&1; echo "rc=$?" >> gpurun_out/j/stress_$i.log
done
