# DES lane-heap drain: parity suites, then event-driven throughput (config2 all-DES, config4 8 scenarios)
python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r2za_pytest.log
LUMOS_FORCE_DES=1 timeout 600 python tools/walk_probe.py config2 1024 2 des_config2 > gpurun_out/r2za_des.log 2>&1
LUMOS_FORCE_DES=1 timeout 900 python tools/walk_probe.py config4 8 1 des_config4_8scen >> gpurun_out/r2za_des.log 2>&1
echo rc=$? >> gpurun_out/r2za_des.log
