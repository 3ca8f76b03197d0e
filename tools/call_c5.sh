python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
( time timeout 2400 python -m pytest tests/test_c5_gpu.py -x -q ) > gpurun_out/c5_tests.log 2>&1; echo "rc=$?" >> gpurun_out/c5_tests.log
timeout 900 python tools/survey.py --configs rand-125M,rmat-50M --algos sssp,bfs,cc,mst --styles vertex,edge,worklist,delta --reps 3 > gpurun_out/survey_c5.log 2>&1
