# Round-end evidence (no full ncu captures: gpurun_out must stay under 64 MiB)
set -x
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_round.json 2> gpurun_out/bench_round.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv \
  --log-file gpurun_out/launches_round.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
timeout 120 python tools/c2_parts.py > gpurun_out/c2_round.json; WL=C1 timeout 120 python tools/c2_parts.py >> gpurun_out/c2_round.json
bash tools/ncu_c2.sh prof_c2_round
