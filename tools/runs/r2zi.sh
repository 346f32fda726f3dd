# host_async e2e + its parity test; final N=1 bench line, reference arm
python -m pytest tests/test_gpu_async.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/r2zi_pytest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2zi_bench.json 2> gpurun_out/r2zi_bench.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2zi_ref.json 2> gpurun_out/r2zi_ref.err
