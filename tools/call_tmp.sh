# WORKLIST local continuation on sparse graphs: parity, timings, C5
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/local5.log 2>&1
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_concurrent_gpu.py -x -q 2>&1 | tail -3 >> gpurun_out/local5.log
echo "== defaults" >> gpurun_out/local5.log
timeout 900 python tools/survey.py --configs grid-24M,rand-25M,rmat-10M --algos sssp,bfs --styles worklist,delta --reps 3 2>&1 | grep -v "^==" >> gpurun_out/local5.log
echo "== C5 defaults" >> gpurun_out/local5.log
timeout 1200 python tools/survey.py --configs rand-125M,rmat-50M --algos sssp,bfs --styles worklist,delta --reps 2 2>&1 | grep -v "^==" >> gpurun_out/local5.log
echo "== C5 local off" >> gpurun_out/local5.log
timeout 1200 python tools/survey.py --configs rand-125M,rmat-50M --algos sssp --styles delta --reps 2 --env FALCON_LOCAL=0 2>&1 | grep -v "^==" >> gpurun_out/local5.log
