python tools/walk_probe.py config5 2048 4 fastpath
python tools/walk_probe.py config4 2048 4 fastpath
python -m pytest tests -m gpu -x -q 2>&1 | tail -4
