python -m pytest tests/test_gpu_estimate.py -m gpu -q -x -k "cluster" 2>&1 | tail -5
python tools/walk_probe.py config3 4096 4 cluster
LUMOS_CLUSTER=0 python tools/walk_probe.py config3 4096 4 coop
