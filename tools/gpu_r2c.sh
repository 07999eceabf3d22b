# C2 kernel v2 (prefix_pair.cu): parity tests, A/B against the round-1 kernel, ncu.
mkdir -p gpurun_out/r2c
timeout 600 python -m pytest tests/test_gpu_lgssm.py -x -q -m gpu > gpurun_out/r2c/pytest_lgssm.log 2>&1; echo "rc=$?" >> gpurun_out/r2c/pytest_lgssm.log
tail -3 gpurun_out/r2c/pytest_lgssm.log
timeout 300 python bench.py --config c2 --no-e2e --no-cpu > gpurun_out/r2c/c2_v2.json 2>&1
AUXMC_PREFIX_V1=1 timeout 300 python bench.py --config c2 --no-e2e --no-cpu --no-check > gpurun_out/r2c/c2_v1.json 2>&1
timeout 300 python bench.py --config c2 --noise rng --no-e2e --no-cpu --no-check > gpurun_out/r2c/c2rng_v2.json 2>&1
for f in c2_v2 c2_v1 c2rng_v2; do python -c "import json,sys; l=json.loads(open('gpurun_out/r2c/$f.json').read().strip().splitlines()[-1]); r=l['roofline']; print('$f', l['value'], l['ms_per_step'], r.get('kernel_ms'), r.get('frac'), l.get('spot_check'))"; done
timeout 600 ncu --set full --import-source on -k regex:k_prefix_pair -c 1 -o gpurun_out/r2c/pair_full python bench.py --config c2 --steps 1 --warmup 1 --no-e2e --no-cpu --no-check > gpurun_out/r2c/ncu.log 2>&1
ls gpurun_out/r2c
