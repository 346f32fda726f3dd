# rebuild path on the GPU: full GPU suite (incl. estimate_whatif parity), config3 bench via rebuild
python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r2zb_pytest.log
python bench.py --config config3 --steps 10 --warmup 3 > gpurun_out/r2zb_bench_config3.json 2> gpurun_out/r2zb_bench_config3.err
