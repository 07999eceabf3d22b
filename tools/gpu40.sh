timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest40.log 2>&1; tail -3 gpurun_out/pytest40.log
timeout 600 python bench.py --sampler dnc --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dnc', d['value'], d['ms_per_step'], d['roofline']['frac'])"
