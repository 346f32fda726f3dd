# K1x source-level profile (config3, one cluster-walk launch)
P="python tools/walk_probe.py config3 4096 1 ncu"
$P > gpurun_out/r3b_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"cluster_walk" -s 1 -c 1 \
    -o gpurun_out/r3b_k1x $P > gpurun_out/r3b_ncu.log 2>&1
echo rc=$? >> gpurun_out/r3b_ncu.log
