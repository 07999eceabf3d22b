timeout 300 python tools/c5_kernels.py 1048576 3
timeout 1500 python -m pytest tests/test_gpu_fixed_point.py tests/test_gpu_lgssm.py tests/test_gpu_tshard.py tests/test_gpu_tshard_aux.py tests/test_gpu_law.py tests/test_gpu_auxk.py tests/test_gpu_shapes.py -q -m gpu 2>&1 | tail -2
