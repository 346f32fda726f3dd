# final code: full GPU suite (release), bounds-checked suite, smoke, bench + reference arm, launch list
python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r2zp_pytest.log
LUMOS_B200_LIB=paper_2504_09307_b200/lib/variants/liblumos_debug.so python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_bounds.py 2>&1 | tail -3 > gpurun_out/r2zp_pytest_bounds.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2zp_smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/r2zp_smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2zp_bench.json 2> gpurun_out/r2zp_bench.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2zp_ref.json 2> gpurun_out/r2zp_ref.err
B="python bench.py --steps 1 --warmup 3 --scenarios 8192 --no-audit --no-cpu-baseline --no-e2e"
$B > gpurun_out/r2zp_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/r2zp_launches.csv $B > gpurun_out/r2zp_ncu1.log 2>&1
