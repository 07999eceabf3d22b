timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest37.log 2>&1; tail -3 gpurun_out/pytest37.log
timeout 900 python bench.py --config c4 --steps 2 --warmup 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', d['value'], d['ms_per_step'], d['roofline']['frac'])"
