mkdir -p gpurun_out/r2x
timeout 600 python -m pytest tests/test_gpu_direct_filter.py -q -m gpu -x 2>&1 | tail -3
timeout 600 python bench.py --config c3 --steps 3 --warmup 1 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3', l['value'], l['ms_per_step'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2x/c3_launches.csv python bench.py --config c3 --T 512 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2x/c3_launches.csv 2>&1 | head -6
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_filter_direct -c 1 -o gpurun_out/r2x/fd_full python bench.py --config c3 --T 256 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r2x/ncu.log 2>&1
