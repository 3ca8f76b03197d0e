# Session 3: BFS VERTEX lazy visited set A/B in warm (survey) conditions, two interleaved passes
set -x
mkdir -p gpurun_out/l
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/l/build.log 2>&1
for p in 1 2; do
  for lz in 256 0; do
    timeout 600 python tools/survey.py --configs rand-25M,rmat-10M,rand-125M,rmat-50M --algos bfs --styles vertex --reps 7 --env FALCON_BFS_LAZY_DIV=$lz > gpurun_out/l/lazy_${lz}_p$p.log 2>&1
  done
done
