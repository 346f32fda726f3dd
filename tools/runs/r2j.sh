python tools/walk_probe.py config5 2048 4 prephilox_track1fast
LUMOS_B200_LIB=paper_2504_09307_b200/lib/variants/liblumos_nopre.so python tools/walk_probe.py config5 2048 4 track1fast_nopre
python tools/walk_probe.py config4 2048 4 prephilox_track1fast
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
