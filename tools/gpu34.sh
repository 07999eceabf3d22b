timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest34.log 2>&1; tail -3 gpurun_out/pytest34.log
timeout 900 python bench.py --sampler dnc > gpurun_out/b34_c2dnc.json 2>&1; tail -1 gpurun_out/b34_c2dnc.json | cut -c1-1500
