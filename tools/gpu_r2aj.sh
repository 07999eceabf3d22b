timeout 600 python -m pytest tests/test_gpu_direct_filter.py tests/test_gpu_lgssm.py tests/test_gpu_tshard_aux.py -q -m gpu 2>&1 | tail -1
python tools/c3_kernels.py 4096 256 3
