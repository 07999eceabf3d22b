timeout 900 python -m pytest tests/test_gpu_direct_filter.py tests/test_gpu_lgssm.py tests/test_gpu_shapes.py tests/test_gpu_auxk.py -q -m gpu -k "not c5" 2>&1 | tail -1
timeout 300 python tools/c3_kernels.py 4096 256 3 | grep -E "step|seq"
