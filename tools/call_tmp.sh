timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "load_flags or load_validation" 2>&1 | tail -1
