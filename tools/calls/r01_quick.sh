# quick GPU check: build, smoke, the fast parity tests, a survey of rand-25M / rmat-10M
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "not full_config and not three_passes" > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python tools/survey.py --configs ${CONFIGS:-rand-25M,rmat-10M} --algos ${ALGOS:-sssp,bfs} --styles ${STYLES:-vertex,edge,worklist} --reps 3 > gpurun_out/survey.log 2>&1
