run() { timeout 600 python tools/survey.py --configs $4 --algos $1 --styles $2 --reps 3 2>&1 | grep -v "==" | sed "s/^/$3 /"; }
for D in 16 32 64 128; do
FALCON_DENSE_DIV=$D run sssp,bfs worklist dense$D rand-25M,rmat-10M,grid-24M
done
