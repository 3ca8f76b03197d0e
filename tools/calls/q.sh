# Quick GPU iteration: build, optional tests ($Q_TESTS), survey ($Q_SURVEY = configs:algos:styles), traces ($Q_TRACES)
set -x
mkdir -p gpurun_out/q
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/q/build.log 2>&1
if [ -n "$Q_TESTS" ]; then timeout 1200 python -m pytest $Q_TESTS -x -q > gpurun_out/q/tests.log 2>&1; echo "rc=$?" >> gpurun_out/q/tests.log; fi
if [ -n "$Q_SURVEY" ]; then IFS=: read c al st <<< "$Q_SURVEY"; timeout 900 python tools/survey.py --configs $c --algos $al --styles $st --reps 5 > gpurun_out/q/survey.log 2>&1; fi
for tr in $Q_TRACES; do IFS=: read c a s <<< "$tr"; FALCON_TRACE=1 timeout 300 python tools/run_one.py --config $c --algo $a --style $s --reps 2 --profile > gpurun_out/q/tr_${c}_${a}_${s}.log 2>&1; done
if [ -n "$Q_CMD" ]; then bash -c "$Q_CMD" > gpurun_out/q/cmd.log 2>&1; fi
