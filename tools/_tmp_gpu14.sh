timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gputest_final.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_final.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_final.json')); r=d['roofline']; print(d['value'], d['ms_per_step'], r['sweep_ms'], r['frac'], r['traffic'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks'])"
