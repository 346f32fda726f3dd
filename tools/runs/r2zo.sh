# DES read-only tables through the non-coherent cache (__ldg): parity + throughput
python -m pytest tests/test_gpu_parity.py tests/test_gpu_metrics.py tests/test_gpu_bounds.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/r2zo_pytest.log
LUMOS_FORCE_DES=1 timeout 600 python tools/walk_probe.py config2 1024 2 des_ldg >> gpurun_out/r2zo_des.log 2>&1
LUMOS_FORCE_DES=1 timeout 600 python tools/walk_probe.py config4 8 1 des_c4_ldg >> gpurun_out/r2zo_des.log 2>&1
LUMOS_FORCE_DES=1 timeout 900 python tools/walk_probe.py config4 256 1 des_c4_256 >> gpurun_out/r2zo_des.log 2>&1
