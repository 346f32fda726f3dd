python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2z_smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/r2z_smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2z_bench.json 2> gpurun_out/r2z_bench.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2z_ref.json 2> gpurun_out/r2z_ref.err
B="python bench.py --steps 1 --warmup 3 --scenarios 8192 --no-audit --no-cpu-baseline --no-e2e"
$B > gpurun_out/r2z_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/r2z_launches.csv $B > gpurun_out/r2z_ncu1.log 2>&1
P="python tools/walk_probe.py config5 2048 1 ncu"
$P > gpurun_out/r2z_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"replay_walk" -s 1 -c 1 \
    -o gpurun_out/r2z_walk $P > gpurun_out/r2z_ncu2.log 2>&1
