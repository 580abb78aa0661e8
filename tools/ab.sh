for L in ab/lib_f4.so ab/lib_f6.so; do echo "== $L"; FDW_LIB=$L timeout 300 python tools/quick_perf.py 2d 2>&1 | grep '"C2"\|C1' | cut -c1-300; done
