# A/B of two library builds on the developed-field C4 step time (same box):
#   bash tools/ab_lib.sh ab/lib_old.so paper_2201_05278_b200/libfdwave_cuda.so
for rep in 1 2 3; do
  for L in "$@"; do
    echo -n "$L rep$rep "; FDW_LIB=$L CASES=exact DEV=${DEV:-1500} T=${T:-1000} timeout 300 python tools/power_probe.py
  done
done
