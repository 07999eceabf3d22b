mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest30.log 2>&1; tail -3 gpurun_out/pytest30.log
timeout 600 python bench.py --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['value'], d['ms_per_step'], d['roofline'])"
timeout 600 python bench.py --no-cpu --no-e2e --noise rng 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2 rng', d['value'], d['ms_per_step'])"
