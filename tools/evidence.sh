# One GPU call: ncu --set full of the current best-style relax kernels on
# rand-25M / rmat-10M (profiling mode: host-driven rounds, so ncu sees them),
# a per-launch L2 / DRAM metric list of each run, per-round traces and a
# survey with stats.  Reports are summarised ON THE BOX (ncu -i) and the
# .ncu-rep files deleted, so gpurun_out/ stays far below gpurun's 64 MiB.
# Usage (under gpurun):  EV_RUNS="tag:config:algo:style:regex:skip:count ..." bash tools/evidence.sh
set -x
O=gpurun_out/ev
mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,lts__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_requests.sum,sm__warps_active.avg.pct_of_peak_sustained_active
run() {   # tag config algo style regex skip count
  timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/$1_launches.csv \
      python tools/run_one.py --config $2 --algo $3 --style $4 --reps 1 --profile > $O/$1_launches.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$5" -s $6 -c $7 \
      -o $O/$1 python tools/run_one.py --config $2 --algo $3 --style $4 --reps 1 --profile > $O/$1.log 2>&1
  if [ -f $O/$1.ncu-rep ]; then
    python tools/ncu_summary.py $O/$1.ncu-rep > $O/$1_summary.txt 2>&1
    python tools/ncu_hot.py $O/$1.ncu-rep 30 > $O/$1_hot.txt 2>&1
    ncu -i $O/$1.ncu-rep --page details > $O/$1_details.txt 2>&1
    rm -f $O/$1.ncu-rep
  fi
}
if [ -n "$EV_TESTS" ]; then
  timeout 900 python -m pytest $EV_TESTS -x -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
fi
if [ -z "$EV_NOSURVEY" ]; then
  timeout 900 python tools/survey.py --configs ${EV_CONFIGS:-rand-25M,rmat-10M} --algos sssp,bfs,cc --styles vertex,edge,worklist,delta --reps 3 > $O/survey.log 2>&1
fi
for tr in $EV_TRACES; do   # config:algo:style
  IFS=: read c a s <<< "$tr"
  FALCON_TRACE=1 timeout 300 python tools/run_one.py --config $c --algo $a --style $s --reps 1 --profile > $O/trace_${c}_${a}_${s}.log 2>&1
done
for r in $EV_RUNS; do
  IFS=: read tag c a s rx sk cn <<< "$r"
  run $tag $c $a $s "$rx" $sk $cn
done
ls -la $O
du -sh gpurun_out
