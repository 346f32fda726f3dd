# GPU suite + smoke on the current code (deadlock witness, DES lane heap, rebuild, scanner)
python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r2zg_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2zg_smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/r2zg_smoke.log
