python tools/c4_kernels.py 1 3
AUXMC_LIB_PATH=tools/_exp/cs16.so python tools/c4_kernels.py 1 3
timeout 600 python -m pytest tests/test_gpu_fkpg.py tests/test_gpu_shapes.py -q -m gpu -k "pit or c4" 2>&1 | tail -1
