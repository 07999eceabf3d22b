mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest15.log 2>&1; tail -3 gpurun_out/pytest15.log
timeout 900 python bench.py --config c3 --T 512 --steps 3 --warmup 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['value'], d['ms_per_step'], 'ms')"
A="bench.py --config c3 --T 16 --chains 148 --steps 1 --warmup 1"
bash tools/prof.sh k_filter_seq prof_c3_filt $A
bash tools/prof.sh k_bwd_elements prof_c3_bwd $A
