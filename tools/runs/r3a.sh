# config3 bench with the proven-window cluster walk; full GPU suite; smoke
python bench.py --config config3 --steps 10 --warmup 3 > gpurun_out/r3a_bench_config3.json 2> gpurun_out/r3a_bench_config3.err
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/r3a_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3a_smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/r3a_smoke.log
