timeout 600 python -m pytest tests/test_gpu_fkpg.py tests/test_gpu_shapes.py tests/test_gpu_pm.py tests/test_gpu_failures.py -q -m gpu 2>&1 | tail -1
timeout 120 python tools/c4_kernels.py 1 3 | head -2
timeout 300 python tools/c4_kernels.py 148 2 | head -2
