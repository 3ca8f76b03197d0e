python tools/e2e_timing.py > gpurun_out/e2e_timing.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_concurrent_gpu.py -x -q -k "not full_config and not three" 2>&1 | tail -1 >> gpurun_out/e2e_timing.log
timeout 600 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/bench_e2e.log 2>&1
