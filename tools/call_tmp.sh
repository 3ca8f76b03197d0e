timeout 1500 python -m pytest tests/test_partition_gpu.py tests/test_partition.py tests/test_c5_gpu.py -x -q 2>&1 | tail -2
