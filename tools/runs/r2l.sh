python tools/walk_probe.py config3 4096 4 coop_minb3
LUMOS_B200_LIB=paper_2504_09307_b200/lib/variants/liblumos_coop2.so python tools/walk_probe.py config3 4096 4 coop_minb2
python -m pytest tests/test_gpu_estimate.py -q -x 2>&1 | tail -2
