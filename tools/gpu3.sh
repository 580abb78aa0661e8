set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -x -q 2>&1 | tail -5
timeout 900 python tools/quick_perf.py 2>&1 | tail -20
./oracle/_ref/test_kernel_cuda 2>&1 | tail -30
