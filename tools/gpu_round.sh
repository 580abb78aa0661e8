# Round-end evidence in one call: GPU suite, smoke, bench line, ncu launch list
# of the bench command, ncu --set full of the TMA sweep (developed field) and
# of one resident 2D chunk (C2).
set -x
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_round.json 2> gpurun_out/bench_round.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv \
  --log-file gpurun_out/launches_round.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
STEPS=2000 PROF=2 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sweep3d_tma -s 2000 -c 1 \
  -o gpurun_out/prof_round python tools/developed.py > gpurun_out/ncu_round.log 2>&1; echo "full rc=$?"
bash tools/ncu_c2.sh prof_c2_round
timeout 120 python tools/c2_parts.py > gpurun_out/c2_round.json; WL=C1 timeout 120 python tools/c2_parts.py >> gpurun_out/c2_round.json
