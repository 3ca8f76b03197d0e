# Round-2 warm traffic table: the same best-style calls as tools/traffic.py, under ncu with
# --cache-control none (L2 contents kept across launches, as in a real run), one metric pass.
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed
timeout 1500 ncu --metrics $M --cache-control none --clock-control none --csv --log-file gpurun_out/traffic_warm.csv python tools/traffic.py run --out gpurun_out/traffic_warm_stats.json > gpurun_out/traffic_warm.log 2>&1
grep -c "pass" gpurun_out/traffic_warm.log
