mkdir -p gpurun_out
timeout 1210 python -m pytest tests -x -q -m gpu > gpurun_out/pytest21.log 2>&1; tail -3 gpurun_out/pytest21.log
timeout 900 python bench.py --config c3 --T 512 --steps 3 --warmup 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['value'], d['ms_per_step'], 'ms')"
C3="python bench.py --config c3 --T 256 --steps 1 --warmup 1"
$C3 > gpurun_out/c3_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 2100 --csv --log-file gpurun_out/c3_launches10.csv $C3 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/c3_launches10.csv 2>&1 | head -6
A="bench.py --config c3 --T 16 --chains 148 --steps 1 --warmup 1"
bash tools/prof.sh k_filter_seq prof_c3_filt7 $A
