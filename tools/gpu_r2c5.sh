timeout 300 python tools/c5_kernels.py 1048576 3 2>&1 | grep -E "iteration|k_pg"
timeout 2400 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
