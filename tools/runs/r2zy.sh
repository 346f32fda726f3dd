# ncu --set full of the event-driven kernel (config 2, every scenario event-driven)
P="python tools/walk_probe.py config2 1024 1 ncu"
LUMOS_FORCE_DES=1 $P > gpurun_out/r2zy_plain.log 2>&1 && \
LUMOS_FORCE_DES=1 ncu --set full --clock-control none --import-source on -k regex:"des_kernel" -s 1 -c 1 \
    -o gpurun_out/r2zy_des $P > gpurun_out/r2zy_ncu.log 2>&1
echo rc=$? >> gpurun_out/r2zy_ncu.log
