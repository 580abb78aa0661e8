set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 900 python tools/quick_perf.py 2>&1 | head -4
