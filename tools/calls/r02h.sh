# Session-3 validation of HEAD: build, smoke, full GPU suite, bench line
set -x
mkdir -p gpurun_out/h
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/h/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/h/smoke.log
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/h/tests.log 2>&1; echo "rc=$?" >> gpurun_out/h/tests.log
timeout 900 python bench.py --out gpurun_out/h/bench.json > gpurun_out/h/bench.log 2>&1; echo "rc=$?" >> gpurun_out/h/bench.log
