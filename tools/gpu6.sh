mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_lgssm.py -x -q -m gpu 2>&1 | tail -3
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, 'Gct/s', d['ms_per_step'], 'ms', d['roofline']['kernel_ms'], d['roofline']['frac'])"
for s in dnc seq; do timeout 600 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu --sampler $s --noise rng 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$s', d['value']/1e9, 'Gct/s', d['ms_per_step'], 'ms')"; done
