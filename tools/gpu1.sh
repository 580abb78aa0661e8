set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -15
timeout 600 python tools/quick_perf.py 2>&1 | tail -20
