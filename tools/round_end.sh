# One GPU call: full GPU tests, smoke, bench line, ncu launch list of one bench
# step, ncu --set full of the dominant relax kernel (rand-25M).
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --out gpurun_out/bench.json > gpurun_out/bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${HOT_KERNEL:-k_edge}" -s ${HOT_SKIP:-13} -c 3 -o gpurun_out/hot python tools/run_one.py --config rand-25M --algo ${HOT_ALGO:-sssp} --style ${HOT_STYLE:-edge} --reps 1 --profile > gpurun_out/ncu_hot.log 2>&1
