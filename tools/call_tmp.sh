timeout 900 python tools/survey.py --configs rand-125M,rmat-50M --algos sssp --styles vertex,worklist,edge --reps 3 2>&1 | grep -v "=="
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "layouts" 2>&1 | tail -1
