# Session 3: EDGE 8-bit sources (v3, raw-word prefetch, 48 regs) timings + parity; stress after the C5 tests
set -x
mkdir -p gpurun_out/k
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/k/build.log 2>&1
timeout 600 python tools/survey.py --configs rand-25M,rmat-10M --algos sssp,bfs --styles edge,vertex,worklist,delta --reps 5 > gpurun_out/k/survey.log 2>&1
timeout 900 python -m pytest tests/test_edge_src8_gpu.py tests/test_parity_gpu.py tests/test_round2_gpu.py tests/test_overflow_gpu.py -q -m gpu > gpurun_out/k/tests.log 2>&1; echo "rc=$?" >> gpurun_out/k/tests.log
for i in 1 2 3; do
  timeout 900 python -m pytest tests/test_c5_gpu.py tests/test_concurrent_gpu.py -x -q > gpurun_out/k/stress_$i.log 2>&1; echo "rc=$?" >> gpurun_out/k/stress_$i.log
done
