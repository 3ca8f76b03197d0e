timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "delta or layouts or repeat" 2>&1 | tail -1
timeout 900 python tools/survey.py --configs rand-25M,rmat-10M,grid-24M,rand-125M --algos sssp --styles delta --reps 3 2>&1 | grep -v "=="
