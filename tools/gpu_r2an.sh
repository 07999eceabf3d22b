timeout 600 python -m pytest tests/test_gpu_direct_filter.py tests/test_gpu_shapes.py -k "direct or c3 or l96 or rank1 or linear or broken" -q -m gpu 2>&1 | tail -2
python tools/c3_kernels.py 4096 256 3 | head -2
AUXMC_LIB_PATH=tools/_exp/fdst.so python tools/fd_stamps.py
