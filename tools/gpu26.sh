mkdir -p gpurun_out
for T in 4096 65536; do
timeout 600 python bench.py --config c5 --T $T --steps 2 --warmup 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 T=$T', d['value'], d['ms_per_step'], 'ms', d['config'].get('accept_rate'))"
done
C5="python bench.py --config c5 --T 16384 --steps 1 --warmup 1"
$C5 > gpurun_out/c5_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/c5_launches.csv $C5 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/c5_launches.csv 2>&1 | head -14
