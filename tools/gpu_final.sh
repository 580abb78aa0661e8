# Round-end evidence: bench line, ncu launch list of the bench command, one
# ncu --set full capture of the TMA sweep on a developed wavefield.
set -x
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv \
  --log-file gpurun_out/launches_final.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
STEPS=2000 PROF=2 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sweep3d_tma -s 2000 -c 1 \
  -o gpurun_out/prof_final python tools/developed.py > gpurun_out/ncu_final.log 2>&1; echo "full rc=$?"
