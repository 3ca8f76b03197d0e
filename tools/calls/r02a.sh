# GPU call: smoke, loopback/partition/overflow tests, bench (single + simulated partition), traffic table
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests/test_loopback_gpu.py tests/test_partition_gpu.py tests/test_overflow_gpu.py -x -q > gpurun_out/tests.log 2>&1; echo rc=$? >> gpurun_out/tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --out gpurun_out/bench.json > gpurun_out/bench.log 2>&1
timeout 300 python bench.py --simulate 4 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --out gpurun_out/bench_sim4.json > gpurun_out/bench_sim4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/traffic.csv python tools/traffic.py run --out gpurun_out/traffic_stats.json > gpurun_out/traffic.log 2>&1
