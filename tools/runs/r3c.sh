# final: full GPU suite, smoke, config5 bench line
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/r3c_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3c_smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/r3c_smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r3c_bench.json 2> gpurun_out/r3c_bench.err
