mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 900 python bench.py --config c3 --T 512 --steps 2 --warmup 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 T=512', d['value'], d['ms_per_step'], 'ms', d['roofline']['frac'])"
timeout 900 python bench.py --config c4 --T 2048 --chains 1 --steps 2 --warmup 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 pit T=2048', d['value'], d['ms_per_step'], 'ms')"
C3="python bench.py --config c3 --T 256 --steps 1 --warmup 1"
$C3 > gpurun_out/c3_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/c3_launches4.csv $C3 > /dev/null 2>&1
