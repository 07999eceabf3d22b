mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
for c in c1 c3; do timeout 600 python bench.py --config $c --steps 5 --warmup 2 2>&1 | tail -1 | cut -c1-600; done
timeout 900 python bench.py --config c4 --steps 2 --warmup 1 --chains 1 2>&1 | tail -1 | cut -c1-500
timeout 900 python bench.py --config c4 --steps 2 --warmup 1 --chains 1 --sampler dnc 2>&1 | tail -1 | cut -c1-500
