python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "not full_config and not three_passes" > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
for Q in 1 0; do
FALCON_WL_NOQ=$Q timeout 900 python tools/survey.py --algos sssp,bfs --styles worklist --reps 3 2>&1 | grep -v "==" | sed "s/^/noq=$Q /"
done > gpurun_out/survey_noq.log
