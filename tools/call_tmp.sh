# BFS VERTEX: bottom-up round inside the expansion kernel (one launch per round) -- parity + timing
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pullmerge.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_concurrent_gpu.py -x -q -k "bfs or small or layouts or golden or run_many" 2>&1 | tail -2 >> gpurun_out/pullmerge.log
timeout 900 python tools/survey.py --configs rand-25M,rmat-10M,grid-24M --algos bfs --styles vertex --reps 5 2>&1 | grep -v "^==" >> gpurun_out/pullmerge.log
