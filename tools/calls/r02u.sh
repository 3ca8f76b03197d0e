# Session 3: BFS WORKLIST bottom-up rounds (persistent-kernel fix) -- full GPU suite, then the bench line
set -x
mkdir -p gpurun_out/u
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/u/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/u/smoke.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/u/tests.log 2>&1; echo "rc=$?" >> gpurun_out/u/tests.log
timeout 900 python bench.py --out gpurun_out/u/bench.json > gpurun_out/u/bench.log 2>&1; echo "rc=$?" >> gpurun_out/u/bench.log
