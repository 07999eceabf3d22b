mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_auxk.py -x -q -m gpu 2>&1 | tail -25
