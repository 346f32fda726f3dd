python tools/walk_probe.py config5 2048 4 u32jitter
python tools/walk_probe.py config4 2048 4 u32jitter
python tools/walk_probe.py config3 4096 4 u32jitter
python -m pytest tests/test_gpu_parity.py tests/test_gpu_walk_variants.py tests/test_golden.py -m gpu -q -x 2>&1 | tail -2
