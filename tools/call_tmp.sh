# local continuation defaults + unit-weight BFS: parity, then timings
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/local4.log 2>&1
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_concurrent_gpu.py -x -q 2>&1 | tail -5 >> gpurun_out/local4.log
echo "== defaults" >> gpurun_out/local4.log
timeout 900 python tools/survey.py --configs grid-24M,rand-25M,rmat-10M --reps 3 2>&1 | grep -v "^==" >> gpurun_out/local4.log
echo "== grid bfs unit LOCAL=64" >> gpurun_out/local4.log
timeout 600 python tools/survey.py --configs grid-24M --algos bfs,sssp --styles worklist,delta --reps 3 --env FALCON_LOCAL=64 2>&1 | grep -v "^==" >> gpurun_out/local4.log
