CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sweep3d_tma -s 20 -c 1 -o gpurun_out/prof_x2 $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
