timeout 600 python -m pytest tests/test_gpu_lgssm.py -x -q -m gpu 2>&1 | tail -2
for i in 1; do timeout 300 python bench.py --config c2 --no-e2e --no-cpu --steps 20 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2', round(l['roofline']['kernel_ms'],4), l['roofline']['frac'], l['spot_check']['max_rel_err'])"; done
AUXMC_LIB_PATH=tools/_exp/x1.so timeout 300 python bench.py --config c2 --no-e2e --no-cpu --no-check --steps 20 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('x1 noio', round(l['roofline']['kernel_ms'],4))"
AUXMC_LIB_PATH=tools/_exp/x9.so python tools/c2_stamps.py | tail -2
