# Round-2 evidence call: smoke, bench line, ncu launch list of one bench step, the traffic table
# (ncu metrics incl. L2 atom/red sectors per best-style call), ncu --set full of the best-style
# kernels' heavy rounds, compute-sanitizer on the tiny config.
set -x
mkdir -p gpurun_out/san gpurun_out/ev
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --out gpurun_out/bench.json > gpurun_out/bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-classes > gpurun_out/launches_bench.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_read.sum,lts__t_sector_hit_rate.pct
timeout 1500 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/traffic.csv python tools/traffic.py run --out gpurun_out/traffic_stats.json > gpurun_out/traffic.log 2>&1
EV_NOSURVEY=1 EV_RUNS="delta:rand-25M:sssp:delta:k_expand_warp:22:3 bfspull:rand-25M:bfs:vertex:k_pull:13:3 bfspush:rand-25M:bfs:vertex:k_expand_warp:11:2 rmatdelta:rmat-10M:sssp:delta:k_expand_warp:25:3 ccwl:rand-25M:cc:worklist:k_cc:0:3" bash tools/evidence.sh
for tool in memcheck racecheck synccheck initcheck; do
  for a in sssp bfs cc; do
    for s in vertex edge worklist; do
      timeout 300 compute-sanitizer --tool $tool --error-exitcode 9 python tools/run_one.py --config tiny --algo $a --style $s --reps 1 --check > gpurun_out/san/${tool}_${a}_${s}.log 2>&1; echo "rc=$?" >> gpurun_out/san/${tool}_${a}_${s}.log
    done
  done
  timeout 300 compute-sanitizer --tool $tool --error-exitcode 9 python tools/run_one.py --config tiny --algo sssp --style delta --reps 1 --check > gpurun_out/san/${tool}_sssp_delta.log 2>&1; echo "rc=$?" >> gpurun_out/san/${tool}_sssp_delta.log
  timeout 300 compute-sanitizer --tool $tool --error-exitcode 9 python tools/run_one.py --config tiny --algo sssp,bfs --style vertex,worklist --reps 1 --profile --check > gpurun_out/san/${tool}_profiled.log 2>&1; echo "rc=$?" >> gpurun_out/san/${tool}_profiled.log
done
grep -l "ERROR SUMMARY: [1-9]\|rc=[1-9]" gpurun_out/san/*.log > gpurun_out/san/flagged.txt
grep -h "ERROR SUMMARY\|RACECHECK SUMMARY" gpurun_out/san/*.log | sort | uniq -c > gpurun_out/san/summary.txt
