# A/B of library builds on the full C4 bench step (device value + sweep ms), alternating
for r in 1 2; do for L in "$@"; do echo "== $L"; FDW_LIB=$L timeout 600 python bench.py --no-cpu --no-e2e --steps 3 2>/dev/null | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['sweep_ms'], d['roofline']['kernel_ms']['inject'], d['clocks']['sm_mhz'])"; done; done
