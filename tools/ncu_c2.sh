# ncu --set full of one resident 2D launch (C2, 100 steps) after a clean run
timeout 120 python tools/c2_parts.py > gpurun_out/c2_plain.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step2d -s 2 -c 1 -o gpurun_out/${1:-prof_c2} python tools/c2_parts.py > gpurun_out/ncu_c2.log 2>&1; echo "ncu rc=$?"
