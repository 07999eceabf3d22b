timeout 300 python tools/c5_kernels.py 1048576 3 2>&1 | grep -E "iteration|reduce_fill"
timeout 1200 python -m pytest tests/test_gpu_lgssm.py tests/test_gpu_fixed_point.py tests/test_gpu_tshard.py tests/test_gpu_tshard_aux.py -q -m gpu -x 2>&1 | tail -2
