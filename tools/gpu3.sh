mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lgssm.py -x -q -m gpu 2>&1 | tail -15
timeout 300 python tools/quick_c2.py 65536 1024 2>&1 | tail -20
