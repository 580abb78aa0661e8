# One ncu --set full capture of the TMA sweep (C4) after the same command ran clean.
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
OUT=${1:-prof_tma}
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sweep3d_tma -s 20 -c 1 -o gpurun_out/$OUT $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
