# Session 3 final evidence, part 1: smoke, traffic tables (cold + warm, copied into profiles/ on the box
# before the bench reads them), bench line, ncu launch list of one bench step.
set -x
F=gpurun_out/final2
mkdir -p $F
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $F/smoke.log 2>&1; echo "rc=$?" >> $F/smoke.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_read.sum,lts__t_sector_hit_rate.pct
timeout 1500 ncu --metrics $M --clock-control none --csv --log-file $F/traffic.csv python tools/traffic.py run --out $F/traffic_stats.json > $F/traffic.log 2>&1
python tools/traffic.py combine $F/traffic.csv $F/traffic_stats.json > $F/r02_traffic.json && cp $F/r02_traffic.json profiles/r02_traffic.json
MW=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed
timeout 1500 ncu --metrics $MW --cache-control none --clock-control none --csv --log-file $F/traffic_warm.csv python tools/traffic.py run --out $F/traffic_warm_stats.json > $F/traffic_warm.log 2>&1
python tools/traffic.py combine $F/traffic_warm.csv $F/traffic_warm_stats.json > $F/r02_traffic_warm.json && cp $F/r02_traffic_warm.json profiles/r02_traffic_warm.json
timeout 900 python bench.py --out $F/bench.json > $F/bench.log 2>&1; echo "rc=$?" >> $F/bench.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $F/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-classes > $F/launches_bench.log 2>&1
