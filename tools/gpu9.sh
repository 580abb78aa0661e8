timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 900 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "rc=$?"; cat gpurun_out/bench.json | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['e2e'], d['roofline']['frac'], d['clocks'])"
