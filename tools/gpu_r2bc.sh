AUXMC_LIB_PATH=tools/_exp/bwst.so python tools/bwd_stamps.py
python tools/c3_kernels.py 4096 256 3 | head -3
timeout 600 python -m pytest tests/test_gpu_direct_filter.py tests/test_gpu_lgssm.py tests/test_gpu_shapes.py -q -m gpu -k "not c5" 2>&1 | tail -1
