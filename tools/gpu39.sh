timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest39.log 2>&1; tail -3 gpurun_out/pytest39.log
timeout 900 python bench.py --config c3 --T 512 --steps 2 --warmup 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['value'], d['ms_per_step'], d['roofline']['frac'])"
timeout 900 python bench.py --config c5 --steps 2 --warmup 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', d['value'], d['ms_per_step'], d['roofline']['frac'])"
