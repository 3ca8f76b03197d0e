timeout 1500 python -m pytest tests -m gpu -x -q -k "not full_config and not c5 and not three" 2>&1 | tail -1
timeout 600 python tools/survey.py --configs rand-25M --algos sssp,bfs --styles vertex,worklist,delta --reps 3 2>&1 | grep -v "=="
