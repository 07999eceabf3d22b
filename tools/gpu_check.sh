# GPU check on a gpurun box: parity suite + one line per bench config.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- bash tools/gpu_check.sh
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for c in "" "--sampler dnc" "--config c1" "--config c3 --T 512" "--config c4" "--config c5"; do
  timeout 900 python bench.py $c --steps 3 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c' or 'c2', '%.4g' % d['value'], d['unit'], 'ms/step %.4g' % d['ms_per_step'], 'roofline frac', d['roofline'].get('frac'))"
done
