# Round-2 evidence on one B200 (run under gpurun): GPU suite, bench line, ncu
# launch list of the same command, one ncu --set full capture of the sweep on a
# developed C4 wavefield.  Each ncu pass runs only after its command exited 0
# without ncu.
set -x
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gputest_r02.log 2>&1; echo "tests rc=$?"
timeout 900 python bench.py > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; echo "bench rc=$?"
timeout 900 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_short.json 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv \
  --log-file gpurun_out/launches_r02.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
bash tools/ncu_dev.sh prof_dev_r02
