FDW_LIB=ab/lib_etaonly.so timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for i in 1 2; do
for L in ab/lib_head.so ab/lib_etaonly.so; do
  echo "== $L"; FDW_LIB=$L timeout 300 python tools/quick_perf.py 2>&1 | sed -n 1p | cut -c1-300
done; done
