cp paper_1903_01665_b200/libfalcon.so /tmp/libfalcon_base.so
for V in base NO_EVICT_LAST NO_EVICT_FIRST; do
if [ $V = base ]; then cp /tmp/libfalcon_base.so paper_1903_01665_b200/libfalcon.so; else cp paper_1903_01665_b200/libfalcon_$V.so paper_1903_01665_b200/libfalcon.so; fi
timeout 600 python tools/survey.py --configs rand-25M,rmat-10M --algos sssp,bfs,cc --styles vertex,edge,worklist --reps 3 2>&1 | grep -v "==" | sed "s/^/$V /"
done > gpurun_out/evict.log
cp /tmp/libfalcon_base.so paper_1903_01665_b200/libfalcon.so
