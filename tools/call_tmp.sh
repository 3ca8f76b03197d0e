python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "not full_config and not three_passes" > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python tools/survey.py --reps 3 > gpurun_out/survey.log 2>&1
timeout 600 python bench.py --out gpurun_out/bench.json > gpurun_out/bench.log 2>&1
