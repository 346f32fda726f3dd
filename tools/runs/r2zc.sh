# K1x occupancy: register cap (MINB 1/6/8 builds) x shared-memory carveout (driver / 100 %)
P="python tools/walk_probe.py config3 4096 4"
for lib in default cmb6 cmb8; do
  for co in -1 100; do
    if [ $lib = default ]; then L=""; else L="LUMOS_B200_LIB=paper_2504_09307_b200/lib/variants/liblumos_$lib.so"; fi
    env $L LUMOS_CLUSTER_CARVEOUT=$co $P ${lib}_co$co >> gpurun_out/r2zc_probe.log 2>&1
  done
done
