timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python tools/c3_kernels.py 4096 256 3 | head -3
