# GPU call (round 2, session 2 start): build, smoke, full GPU tests, bench line,
# compute-sanitizer on the tiny config, per-round traces of the best styles.
set -x
mkdir -p gpurun_out/san gpurun_out/tr
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --out gpurun_out/bench.json > gpurun_out/bench.log 2>&1
for tr in rand-25M:sssp:delta rand-25M:sssp:worklist rand-25M:bfs:vertex rand-25M:cc:worklist rmat-10M:sssp:vertex rmat-10M:bfs:vertex rmat-10M:cc:worklist; do
  IFS=: read c a s <<< "$tr"
  FALCON_TRACE=1 timeout 300 python tools/run_one.py --config $c --algo $a --style $s --reps 2 --profile > gpurun_out/tr/${c}_${a}_${s}.log 2>&1
done
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
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
grep -h "ERROR SUMMARY" gpurun_out/san/*.log | sort | uniq -c > gpurun_out/san/summary.txt
