python bench.py --steps 10 --warmup 3 > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err
B="python bench.py --steps 1 --warmup 3 --scenarios 8192 --no-audit --no-cpu-baseline --no-e2e"
$B > gpurun_out/r2k_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/r2k_launches.csv $B > gpurun_out/r2k_ncu1.log 2>&1
P="python tools/walk_probe.py config5 2048 1 ncu"
$P > gpurun_out/r2k_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"replay_walk|rank_reduce" -s 2 -c 2 \
    -o gpurun_out/r2k_prof $P > gpurun_out/r2k_ncu2.log 2>&1
