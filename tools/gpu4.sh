set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_known_answers.py -x -q -m gpu 2>&1 | tail -4
timeout 900 python tools/quick_perf.py 2>&1 | tail -20
./oracle/_ref/test_kernel_cuda 2>&1 | grep -E "FAILED|Failure|tests," -A3 | head -20
