timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest35.log 2>&1; tail -3 gpurun_out/pytest35.log
timeout 600 python bench.py --config c1 --steps 50 --warmup 5 2>&1 | tail -1 | cut -c1-900
timeout 600 python bench.py --config c1 --steps 50 --warmup 5 --no-graph 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('eager', d['value'], d['ms_per_step'], d['gpu_launches'])"
