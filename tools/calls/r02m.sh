# Session 3: same-box A/B of the d2ce60d library (before the lazy BFS visited set) against HEAD
set -x
mkdir -p gpurun_out/m
L=paper_1903_01665_b200/libfalcon.so
cp $L build/new.so
for p in 1 2; do
  cp build/old/libfalcon_d2ce60d.so $L
  timeout 600 python tools/survey.py --configs rand-25M,rmat-10M --algos bfs,sssp --styles vertex,delta --reps 7 > gpurun_out/m/old_p$p.log 2>&1
  cp build/new.so $L
  timeout 600 python tools/survey.py --configs rand-25M,rmat-10M --algos bfs,sssp --styles vertex,delta --reps 7 > gpurun_out/m/new_p$p.log 2>&1
done
cp build/new.so $L
