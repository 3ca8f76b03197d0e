# Session 3: memcheck the run_many failure, full GPU suite (no -x), EDGE timings with 8-bit sources
set -x
mkdir -p gpurun_out/i
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/i/build.log 2>&1
timeout 600 compute-sanitizer --tool memcheck python -m pytest tests/test_concurrent_gpu.py -x -q -k "all_jobs" > gpurun_out/i/memcheck_concurrent.log 2>&1; echo "rc=$?" >> gpurun_out/i/memcheck_concurrent.log
timeout 300 python tools/survey.py --configs rand-25M,rmat-10M --algos sssp,bfs --styles edge --reps 5 > gpurun_out/i/survey_edge.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/i/tests.log 2>&1; echo "rc=$?" >> gpurun_out/i/tests.log
