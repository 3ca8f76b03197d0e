timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "memory_cache or golden" 2>&1 | tail -2
