timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python tools/c5_kernels.py | head -3
