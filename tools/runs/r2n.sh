python -m pytest tests/test_gpu_estimate.py -m gpu -q -x -k split_accounting 2>&1 | grep -E "Error|assert|where|^E " | head -40
