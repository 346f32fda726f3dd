# DES breakdown: sorted per-stream runs merged instead of heap-sorted (parity + throughput)
python -m pytest tests/test_gpu_parity.py tests/test_gpu_metrics.py tests/test_gpu_bounds.py tests/test_gpu_async.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/r2zw_pytest.log
LUMOS_FORCE_DES=1 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "event_driven or random or golden or config1" 2>&1 | tail -2 >> gpurun_out/r2zw_pytest.log
LUMOS_FORCE_DES=1 timeout 600 python tools/walk_probe.py config2 1024 2 des_c2 >> gpurun_out/r2zw_des.log 2>&1
LUMOS_FORCE_DES=1 timeout 600 python tools/walk_probe.py config4 8 1 des_c4 >> gpurun_out/r2zw_des.log 2>&1
