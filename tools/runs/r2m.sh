python tools/walk_probe.py config3 4096 4 coop_split_acct
python tools/walk_probe.py config5 2048 2 c5
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
LUMOS_B200_LIB=paper_2504_09307_b200/lib/variants/liblumos_debug.so python -m pytest tests/test_gpu_estimate.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
