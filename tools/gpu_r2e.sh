# C2: log-depth carry pass
mkdir -p gpurun_out/r2e
timeout 600 python -m pytest tests/test_gpu_lgssm.py -x -q -m gpu 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --config c2 --no-e2e --no-cpu --steps 20 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2', round(l['roofline']['kernel_ms'],4), l['roofline']['frac'], l['spot_check']['max_rel_err'])"; done
timeout 300 python bench.py --config c2 --noise rng --no-e2e --no-cpu --no-check --steps 20 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2rng', round(l['roofline']['kernel_ms'],4))"
