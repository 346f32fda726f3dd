# round-2 measurement: full bench line (audit + CPU baseline), then one ncu --set full of K1
python bench.py --steps 10 --warmup 3 > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err
python tools/walk_probe.py config5 2048 1 ncu > gpurun_out/r2d_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:replay_walk -s 1 -c 1 \
    -o gpurun_out/r2d_walk python tools/walk_probe.py config5 2048 1 ncu > gpurun_out/r2d_ncu.log 2>&1
