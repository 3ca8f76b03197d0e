python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -k "not full_config" > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python tools/concurrency.py --configs rand-25M,rmat-10M,grid-24M --reps 3 > gpurun_out/concurrency.log 2>&1
timeout 600 python tools/survey.py --configs rand-25M --reps 3 > gpurun_out/survey.log 2>&1
