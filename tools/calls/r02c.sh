# GPU call: sections / two-graph tests, compute-sanitizer on the tiny config, loopback + parity spot checks
set -x
mkdir -p gpurun_out/san
timeout 900 python -m pytest tests/test_sections_gpu.py tests/test_loopback_gpu.py -x -q > gpurun_out/tests_c.log 2>&1; echo rc=$? >> gpurun_out/tests_c.log
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
