python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "event_driven_path_equals_walk" 2>&1 | tail -2
LUMOS_FORCE_DES=1 timeout 300 python tools/walk_probe.py config2 1024 2 des_config2
LUMOS_FORCE_DES=1 timeout 600 python tools/walk_probe.py config4 296 1 des_config4
LUMOS_FORCE_DES=1 timeout 900 python tools/walk_probe.py config5 148 1 des_config5
