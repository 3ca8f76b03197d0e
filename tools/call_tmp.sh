# adaptive-Δ growth cap x local budget on the grid (and rand / rmat at the default budget)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/dcap.log 2>&1
for C in 32 128 512 4096; do for L in 16 64; do
  echo "== DELTA_CAP=$C LOCAL=$L" >> gpurun_out/dcap.log
  timeout 600 python tools/survey.py --configs grid-24M --algos sssp,bfs --styles worklist,delta --reps 3 --env FALCON_DELTA_CAP=$C FALCON_LOCAL=$L 2>&1 | grep -v "^==" | grep "delta\|bfs" >> gpurun_out/dcap.log
done; done
for C in 32 512; do
  echo "== DELTA_CAP=$C rand/rmat" >> gpurun_out/dcap.log
  timeout 600 python tools/survey.py --configs rand-25M,rmat-10M --algos sssp --styles delta --reps 3 --env FALCON_DELTA_CAP=$C 2>&1 | grep -v "^==" >> gpurun_out/dcap.log
done
