mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -25
timeout 600 python bench.py --steps 10 --warmup 3 2>&1 | tail -3
