# K1x cluster scheduling policy x register cap
P="python tools/walk_probe.py config3 4096 4"
V8="LUMOS_B200_LIB=paper_2504_09307_b200/lib/variants/liblumos_cmb8.so"
for pol in 0 2; do
  env LUMOS_CLUSTER_POLICY=$pol $P pol$pol >> gpurun_out/r2ze_probe.log 2>&1
  env $V8 LUMOS_CLUSTER_POLICY=$pol $P cmb8_pol$pol >> gpurun_out/r2ze_probe.log 2>&1
  env $V8 LUMOS_CLUSTER_POLICY=$pol LUMOS_CLUSTER_CARVEOUT=100 $P cmb8_co100_pol$pol >> gpurun_out/r2ze_probe.log 2>&1
done
Q="python tools/walk_probe.py config3 4096 1 ncu"
for v in default cmb8; do
  if [ $v = default ]; then L=""; else L="$V8"; fi
  env $L LUMOS_CLUSTER_CARVEOUT=100 ncu --section LaunchStats --section Occupancy --metrics sm__cycles_active.min,sm__cycles_active.avg,sm__cycles_active.max,sm__warps_active.avg.per_cycle_active,sm__inst_issued.avg.pct_of_peak_sustained_active,gpu__time_duration.sum --clock-control none -k regex:"cluster_walk" -s 1 -c 1 --csv --page raw $Q > gpurun_out/r2ze_ncu_$v.csv 2> gpurun_out/r2ze_ncu_$v.err
done
