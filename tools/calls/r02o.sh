# Session 3: re-tune with the fixed k_pull / skip_now (same box, survey = warm L2 like bench.py)
set -x
mkdir -p gpurun_out/o
for p in 1 2; do
  for lz in 0 64 256 1024; do
    timeout 600 python tools/survey.py --configs rand-25M,rmat-10M,rand-125M,rmat-50M --algos bfs --styles vertex --reps 5 --env FALCON_BFS_LAZY_DIV=$lz > gpurun_out/o/lazy_${lz}_p$p.log 2>&1
  done
done
for dd in 16 32 64; do
  timeout 600 python tools/survey.py --configs rand-25M,rmat-10M --algos sssp --styles vertex,worklist,delta --reps 5 --env FALCON_DENSE_DIV=$dd > gpurun_out/o/dense_${dd}.log 2>&1
done
for bd in 4 16; do
  timeout 600 python tools/survey.py --configs rand-25M --algos sssp --styles vertex,worklist,delta --reps 5 --env FALCON_BLOCK_DIV=$bd > gpurun_out/o/blk_${bd}.log 2>&1
done
