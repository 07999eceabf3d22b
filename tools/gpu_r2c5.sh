timeout 300 python tools/c5_kernels.py 1048576 3 2>&1 | head -30
timeout 2400 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
