LUMOS_B200_LIB=paper_2504_09307_b200/lib/variants/liblumos_debug.so python -m pytest tests -m gpu -q -x 2>&1 | tail -6
python -m pytest tests/test_gpu_bounds.py -q 2>&1 | tail -4
