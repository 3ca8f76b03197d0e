# GPU call: parity of the DELTA split / pull changes; sweeps
set -x
timeout 1500 python -m pytest tests/test_loopback_gpu.py -x -q > gpurun_out/tests_lb.log 2>&1; echo rc=$? >> gpurun_out/tests_lb.log
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "delta or noq or golden or tiny or star or layouts" > gpurun_out/tests_b.log 2>&1; echo rc=$? >> gpurun_out/tests_b.log
for sd in 0 4 8 16; do
  FALCON_SPLIT_DIV=$sd timeout 600 python tools/survey.py --configs rand-25M,rmat-10M,grid-24M --algos sssp --styles delta --reps 3 > gpurun_out/split_$sd.log 2>&1
done
timeout 600 python tools/survey.py --configs rand-25M,rmat-10M,grid-24M --algos bfs --styles vertex,worklist --reps 3 > gpurun_out/bfs.log 2>&1
FALCON_TRACE=1 FALCON_SPLIT_DIV=8 timeout 300 python tools/run_one.py --config rand-25M --algo sssp --style delta --reps 1 --profile > gpurun_out/trace_delta_split8.log 2>&1
FALCON_TRACE=1 timeout 300 python tools/run_one.py --config rand-25M --algo bfs --style vertex --reps 1 --profile > gpurun_out/trace_bfs.log 2>&1
