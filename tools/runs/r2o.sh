python -m pytest tests -m gpu -q 2>&1 | tail -3
LUMOS_B200_LIB=paper_2504_09307_b200/lib/variants/liblumos_debug.so python -m pytest tests -m gpu -q -x 2>&1 | tail -2
