python -m pytest tests -m gpu -q 2>&1 | tail -3
LUMOS_B200_LIB=paper_2504_09307_b200/lib/variants/liblumos_debug.so python -m pytest tests -m gpu -q -x 2>&1 | tail -2
LUMOS_B200_LIB=paper_2504_09307_b200/lib/variants/liblumos_cl8.so python tools/walk_probe.py config3 4096 4 cluster_minb8
python tools/walk_probe.py config3 4096 4 cluster_default
