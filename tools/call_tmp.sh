for P in 0 1; do
FALCON_PERSIST=$P timeout 900 python tools/survey.py --configs grid-24M,rand-25M --algos sssp,bfs --styles worklist,delta --reps 3 2>&1 | grep -v "==" | sed "s/^/persist=$P /"
done
FALCON_PERSIST=1 FALCON_PERSIST_MAX=16384 timeout 900 python tools/survey.py --configs grid-24M --algos sssp,bfs --styles worklist,delta --reps 3 2>&1 | grep -v "==" | sed "s/^/persist16k /"
