timeout 600 python -m pytest tests/test_gpu_direct_filter.py -q -m gpu 2>&1 | tail -3
python tools/c3_kernels.py 4096 256 3 | head -3
AUXMC_LIB_PATH=tools/_exp/fdl.so python tools/c3_kernels.py 4096 256 3 | head -3
AUXMC_LIB_PATH=tools/_exp/fdst.so python tools/fd_stamps.py
AUXMC_LIB_PATH=tools/_exp/fdstl.so python tools/fd_stamps.py
