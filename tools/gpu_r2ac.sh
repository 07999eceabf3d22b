mkdir -p gpurun_out/r2ac
timeout 600 python -m pytest tests/test_gpu_direct_filter.py tests/test_gpu_lgssm.py -q -m gpu --tb=short 2>&1 | grep -E "Error|error|assert|passed|failed" | head -20
timeout 900 python -m pytest tests/test_gpu_shapes.py -q -m gpu -x -k c3 2>&1 | tail -1
timeout 600 python bench.py --config c3 --steps 3 --warmup 1 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3', l['value'], l['ms_per_step'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2ac/c3_launches.csv python bench.py --config c3 --T 512 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2ac/c3_launches.csv 2>&1 | head -6
