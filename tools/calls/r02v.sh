# Session 3: ncu launch list of one bench step on the final build (after bfs_wl_pull)
set -x
mkdir -p gpurun_out/v
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/v/build.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/v/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-classes > gpurun_out/v/launches_bench.log 2>&1
echo "rc=$?" >> gpurun_out/v/launches_bench.log
