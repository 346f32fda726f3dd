# K1x with 64-thread rank CTAs (LUMOS_CLUSTER_T=64): parity + config3 A/B
LUMOS_CLUSTER_T=64 python -m pytest tests/test_gpu_estimate.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/r2zr_pytest.log
for t in 128 64; do LUMOS_CLUSTER_T=$t python tools/walk_probe.py config3 4096 4 t$t >> gpurun_out/r2zr_probe.log 2>&1; done
for t in 128 64; do LUMOS_CLUSTER_T=$t python tools/walk_probe.py config3 4096 4 t${t}_again >> gpurun_out/r2zr_probe.log 2>&1; done
