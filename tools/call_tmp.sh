timeout 1500 python -m pytest tests/test_partition_gpu.py tests/test_partition.py -x -q 2>&1 | tail -3
for E in 1 2 0; do
FALCON_EXCHANGE=$E timeout 600 python bench.py --mode partition --simulate 8 --config rand-25M --steps 2 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('exchange=$E', round(d['value'],2), 'GTEPS', round(d['ms_per_step'],1), 'ms/step', {k: round(v['ms'],1) for k,v in d['per_run'].items()})"
done
