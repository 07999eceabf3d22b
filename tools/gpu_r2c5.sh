timeout 300 python tools/c3_kernels.py 4096 256 3 2>&1 | head -8
timeout 300 python tools/c5_kernels.py 1048576 3 2>&1 | grep -E "iteration|k_gamma"
timeout 2400 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
