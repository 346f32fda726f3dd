python tools/walk_probe.py config3 4096 4 coop_fastpath
LUMOS_FORCE_DES=1 timeout 600 python tools/walk_probe.py config2 1024 2 des_config2
LUMOS_FORCE_DES=1 timeout 900 python tools/walk_probe.py config4 8 1 des_config4_8scen
python -m pytest tests/test_gpu_estimate.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
