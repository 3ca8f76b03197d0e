# Session 3: k_pull back at 32 registers (8 CTAs/SM) -- same-box A/B against the d2ce60d library
set -x
mkdir -p gpurun_out/n
L=paper_1903_01665_b200/libfalcon.so
cp $L build/new.so
for p in 1 2; do
  cp build/old/libfalcon_d2ce60d.so $L
  timeout 600 python tools/survey.py --configs rand-25M,rmat-10M,rand-125M,rmat-50M --algos bfs --styles vertex --reps 7 > gpurun_out/n/old_p$p.log 2>&1
  cp build/new.so $L
  timeout 600 python tools/survey.py --configs rand-25M,rmat-10M,rand-125M,rmat-50M --algos bfs --styles vertex --reps 7 > gpurun_out/n/new_p$p.log 2>&1
done
cp build/new.so $L
