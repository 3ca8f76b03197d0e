timeout 600 python bench.py --out gpurun_out/bench.json > gpurun_out/bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/launches_bench.log 2>&1
timeout 600 python tools/e2e_timing.py > gpurun_out/e2e_timing.log 2>&1
