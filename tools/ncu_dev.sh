# ncu --set full of one TMA sweep launch on a developed C4 wavefield (step 2000)
STEPS=${STEPS:-2000}
STEPS=$STEPS PROF=20 python tools/developed.py > gpurun_out/dev_plain.log 2>&1 || exit 1
STEPS=$STEPS PROF=2 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sweep3d_tma -s $STEPS -c 1 -o gpurun_out/${1:-prof_dev} python tools/developed.py > gpurun_out/ncu_dev.log 2>&1; echo "ncu rc=$?"
