python -m pytest tests -m gpu -q 2>&1 | tail -3
LUMOS_B200_LIB=paper_2504_09307_b200/lib/variants/liblumos_debug.so python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python bench.py --config config3 --steps 10 --warmup 3 > gpurun_out/r2v_bench_config3.json 2> gpurun_out/r2v_bench_config3.err
python bench.py --config config4 --steps 5 --warmup 3 --no-audit > gpurun_out/r2v_bench_config4.json 2> gpurun_out/r2v_bench_config4.err
