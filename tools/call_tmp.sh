timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "not full_config and not three" 2>&1 | tail -1
timeout 900 python tools/survey.py --configs rand-25M,rmat-10M,grid-24M --algos sssp,bfs --styles vertex,worklist,delta --reps 3 2>&1 | grep -v "=="
