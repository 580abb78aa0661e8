# A/B of two library builds on the C4 sweep (alternating runs, same box)
for r in 1 2; do for L in "$@"; do echo "== $L"; FDW_LIB=$L timeout 300 python tools/quick_perf.py c4only 2>&1 | cut -c1-400; done; done
