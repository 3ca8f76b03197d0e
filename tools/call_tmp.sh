cp paper_1903_01665_b200/libfalcon.so /tmp/libfalcon_pf.so
for V in pf nopf; do
cp /tmp/libfalcon_pf.so paper_1903_01665_b200/libfalcon.so
[ $V = nopf ] && cp paper_1903_01665_b200/libfalcon_nopf.so paper_1903_01665_b200/libfalcon.so
timeout 600 python tools/survey.py --algos sssp,bfs --styles edge --reps 3 2>&1 | grep -v "==" | sed "s/^/$V /"
done
cp /tmp/libfalcon_pf.so paper_1903_01665_b200/libfalcon.so
timeout 900 python -m pytest tests -m gpu -x -q -k "not full_config and not three_passes" 2>&1 | tail -1
