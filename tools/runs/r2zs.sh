# final verification: full GPU suite + smoke on the final commit
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/r2zs_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2zs_smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/r2zs_smoke.log
