timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python bench.py --config c1 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c1', l['value'], l['ms_per_step'], l['gpu_launches']/l['steps'])"
timeout 300 python bench.py --config c5 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c5', l['value'], l['ms_per_step'])"
timeout 300 python tools/c3_kernels.py 4096 256 3 | head -1
