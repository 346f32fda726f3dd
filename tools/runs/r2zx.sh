# final commit: full GPU suite (release + bounds-checked), smoke
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/r2zx_pytest.log
LUMOS_B200_LIB=paper_2504_09307_b200/lib/variants/liblumos_debug.so python -m pytest tests -m gpu -q --deselect tests/test_gpu_bounds.py 2>&1 | tail -3 > gpurun_out/r2zx_pytest_bounds.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2zx_smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/r2zx_smoke.log
