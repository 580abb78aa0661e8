set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
bash tools/ab_env.sh FDW_TMA_PERSIST "1 0"
