timeout 900 python -m pytest tests -m gpu -x -q -k "not full_config" 2>&1 | tail -1
timeout 600 python tools/survey.py --algos cc --reps 5 2>&1 | grep -v "=="
