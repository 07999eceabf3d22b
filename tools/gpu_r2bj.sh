timeout 900 python -m pytest tests/test_gpu_direct_filter.py tests/test_gpu_lgssm.py tests/test_gpu_shapes.py tests/test_gpu_failures.py tests/test_gpu_law.py -q -m gpu -k "not c5" 2>&1 | tail -2
timeout 300 python tools/c3_kernels.py 4096 256 3 | head -3
AUXMC_LIB_PATH=tools/_exp/bwst.so timeout 300 python tools/bwd_stamps.py
