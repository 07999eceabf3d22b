timeout 600 python -m pytest tests/test_gpu_direct_filter.py tests/test_gpu_shapes.py -q -m gpu -k "not c5" 2>&1 | tail -1
python tools/c3_kernels.py 4096 256 3 | head -3
AUXMC_LIB_PATH=tools/_exp/fd0.so python tools/c3_kernels.py 4096 256 3 | head -3
AUXMC_LIB_PATH=tools/_exp/fdst.so python tools/fd_stamps.py | head -4
