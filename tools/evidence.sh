# One GPU call: ncu --set full of the current best-style relax kernels on
# rand-25M / rmat-10M (profiling mode: host-driven rounds, so ncu sees them),
# plus a per-launch L2 / DRAM metric list of each run and a survey with stats.
# Usage (under gpurun):  bash tools/evidence.sh
set -x
mkdir -p gpurun_out/ev
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,lts__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_requests.sum
run() {   # $1 = tag, $2 = config, $3 = algo, $4 = style, $5 = kernel regex, $6 = skip, $7 = count
  timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/ev/$1_launches.csv \
      python tools/run_one.py --config $2 --algo $3 --style $4 --reps 1 --profile > gpurun_out/ev/$1_launches.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$5" -s $6 -c $7 \
      -o gpurun_out/ev/$1 python tools/run_one.py --config $2 --algo $3 --style $4 --reps 1 --profile \
      > gpurun_out/ev/$1.log 2>&1
}
timeout 900 python tools/survey.py --configs rand-25M,rmat-10M --algos sssp,bfs,cc --styles vertex,edge,worklist,delta --reps 3 > gpurun_out/ev/survey.log 2>&1
run sssp_wl_rand rand-25M sssp worklist k_expand_warp 14 2
run sssp_v_rand rand-25M sssp vertex k_expand_warp 14 2
run sssp_d_rand rand-25M sssp delta k_expand_warp 40 2
run bfs_v_rand rand-25M bfs vertex "k_expand_warp|k_pull" 14 6
run sssp_v_rmat rmat-10M sssp vertex k_expand_warp 10 2
run bfs_v_rmat rmat-10M bfs vertex "k_expand_warp|k_pull" 8 6
ls -la gpurun_out/ev
