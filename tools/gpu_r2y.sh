mkdir -p gpurun_out/r2y
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2y/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2y/pytest_gpu.log
tail -5 gpurun_out/r2y/pytest_gpu.log
timeout 600 python bench.py --config c3 --steps 3 --warmup 1 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3', l['value'], l['ms_per_step'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2y/c3_launches.csv python bench.py --config c3 --T 512 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2y/c3_launches.csv 2>&1 | head -8
