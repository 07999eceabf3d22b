mkdir -p gpurun_out/r2ag
timeout 600 python -m pytest tests/test_gpu_direct_filter.py -q -m gpu --tb=short 2>&1 | grep -E "Error|error|assert|passed|failed" | head -20
timeout 900 python -m pytest tests/test_gpu_shapes.py -q -m gpu -x -k c3 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2ag/c3_launches.csv python bench.py --config c3 --T 512 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2ag/c3_launches.csv 2>&1 | head -4
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_filter_direct -c 1 -o gpurun_out/r2ag/fd_full python bench.py --config c3 --T 256 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r2ag/ncu.log 2>&1
