# K1x without the per-finish wrap check when the host proves the uint32 window
python -m pytest tests/test_gpu_estimate.py tests/test_gpu_bounds.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/r2zz_pytest.log
for pol in 0 2; do for k in 1 2; do LUMOS_CLUSTER_POLICY=$pol python tools/walk_probe.py config3 4096 4 nochk_pol${pol}_$k >> gpurun_out/r2zz_probe.log 2>&1; done; done
