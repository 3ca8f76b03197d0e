# grid-24M DELTA / BFS WORKLIST per-round trace with and without local continuation (host-driven profiling mode)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/trace.log 2>&1
for L in 0 16; do
  echo "== FALCON_LOCAL=$L (BFS unit-weight Δ-stepping needs local on)" >> gpurun_out/trace.log
  FALCON_LOCAL=$L FALCON_TRACE=1 timeout 600 python tools/run_one.py --config grid-24M --algo sssp,bfs --style delta,worklist --reps 1 --profile > gpurun_out/trace_$L.out 2> gpurun_out/trace_$L.err
  grep "rep0" gpurun_out/trace_$L.out >> gpurun_out/trace.log
done
