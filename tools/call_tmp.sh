python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests/test_mst_gpu.py -x -q > gpurun_out/mst_tests.log 2>&1; echo "rc=$?" >> gpurun_out/mst_tests.log
timeout 900 python tools/survey.py --algos mst --styles vertex,edge --reps 3 > gpurun_out/survey_mst.log 2>&1
