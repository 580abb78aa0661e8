# A/B of a presence flag (set vs unset) on the developed-field C4 step time:
#   bash tools/ab_flag.sh FDW_NO_FUSED_INJECT
VAR=$1
for rep in 1 2 3; do
  echo -n "unset rep$rep "; env -u $VAR CASES=exact DEV=${DEV:-1500} T=${T:-1000} timeout 300 python tools/power_probe.py
  echo -n "$VAR=1 rep$rep "; env $VAR=1 CASES=exact DEV=${DEV:-1500} T=${T:-1000} timeout 300 python tools/power_probe.py
done
