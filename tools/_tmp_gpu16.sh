timeout 600 python tools/quick_perf.py f64 2>&1 | cut -c1-330
FDW_TMA_PD64=1 timeout 600 python tools/quick_perf.py f64 2>&1 | head -1 | cut -c1-330
FDW_TMA_PD64=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_guards.py -q -x -k "float64 or double or f64 or 3d" > gpurun_out/pd64_tests.log 2>&1; echo "pd64 tests rc=$?"; tail -2 gpurun_out/pd64_tests.log
