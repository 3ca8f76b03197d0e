timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
python tools/survey.py --configs rand-25M,rmat-10M,grid-24M --reps 3 > gpurun_out/survey.log 2>&1
python tools/e2e_timing.py > gpurun_out/e2e_timing.log 2>&1
timeout 600 python bench.py --out gpurun_out/bench.json > gpurun_out/bench.log 2>&1
