# DES with lane state in shared memory: parity suites touching the event-driven path, throughput A/B
python -m pytest tests/test_gpu_parity.py tests/test_gpu_metrics.py tests/test_gpu_retime.py tests/test_gpu_bounds.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/r2zn_pytest.log
LUMOS_FORCE_DES=1 LUMOS_FORCE_DES=1 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "event_driven or random or golden or config1" 2>&1 | tail -2 >> gpurun_out/r2zn_pytest.log
for m in 1 0; do
  LUMOS_DES_SMEM=$m LUMOS_FORCE_DES=1 timeout 600 python tools/walk_probe.py config2 1024 2 des_smem$m >> gpurun_out/r2zn_des.log 2>&1
  LUMOS_DES_SMEM=$m LUMOS_FORCE_DES=1 timeout 600 python tools/walk_probe.py config4 8 1 des_c4_smem$m >> gpurun_out/r2zn_des.log 2>&1
done
