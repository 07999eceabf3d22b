timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python bench.py --config c4 --chains 1 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c4 1 chain', l['ms_per_step'], l['value'])"
timeout 600 python bench.py --config c4 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c4 148 chains', l['ms_per_step'], l['value'], l['roofline']['frac'])"
