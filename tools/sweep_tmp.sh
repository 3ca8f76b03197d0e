for BD in 8 2; do
echo "## BLOCK_DIV=$BD"
FALCON_BLOCK_DIV=$BD python tools/survey.py --configs rand-25M,rmat-10M,grid-24M --algos sssp,bfs --styles vertex,edge,worklist --reps 3 2>&1 | grep -v "^=="
done
