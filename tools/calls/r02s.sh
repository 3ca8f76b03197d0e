# Session 3 final evidence, part 2: ncu --set full of the best-style relax kernels (and SSSP EDGE, the bench
# line's dominant kernel), survey of all five configs, the full GPU suite.
set -x
F=gpurun_out/final2
mkdir -p $F
python -c "import __graft_entry__ as g; g.build()" > $F/build2.log 2>&1
timeout 2000 python -m pytest tests -q -m gpu > $F/tests.log 2>&1; echo "rc=$?" >> $F/tests.log
EV_NOSURVEY=1 EV_RUNS="delta:rand-25M:sssp:delta:k_expand_warp:22:3 edge:rand-25M:sssp:edge:k_edge:14:3 bfspull:rand-25M:bfs:vertex:k_pull:13:3 bfspush:rand-25M:bfs:vertex:k_expand_warp:11:2 rmatdelta:rmat-10M:sssp:delta:k_expand_warp:25:3 rmatbfs:rmat-10M:bfs:vertex:k_pull:5:3 ccwl:rand-25M:cc:worklist:k_cc:0:3" bash tools/evidence.sh
rm -rf $F/ev; mv gpurun_out/ev $F/ev
timeout 900 python tools/survey.py --configs rand-25M,rmat-10M,grid-24M,rand-125M,rmat-50M --reps 5 > $F/survey.log 2>&1
du -sh gpurun_out
