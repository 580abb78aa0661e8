# A/B of an environment knob on the developed-field C4 step time and on one
# sweep's DRAM bytes:  bash tools/ab_env.sh VAR "v1 v2 ..."
VAR=$1; VALS=$2
for rep in 1 2; do
  for v in $VALS; do
    echo -n "$VAR=$v rep$rep "; env $VAR=$v CASES=exact DEV=${DEV:-1500} T=${T:-1000} timeout 300 python tools/power_probe.py
  done
done
for v in $VALS; do
  env $VAR=$v ZS=6 timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:sweep3d_tma -s 1 -c 1 --csv python tools/zseg_traffic.py 2>/dev/null | grep -E '"(dram|gpu|lts)' | awk -F'","' -v t="$VAR=$v" '{print t, $(NF-2), $NF}'
done
