mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/b32_c2.json 2> gpurun_out/b32_c2.err
timeout 900 python bench.py --impl reference > gpurun_out/b32_ref.json 2> gpurun_out/b32_ref.err
timeout 600 python bench.py --sampler dnc --no-cpu > gpurun_out/b32_c2dnc.json 2>&1
timeout 600 python bench.py --config c1 --steps 20 --warmup 5 > gpurun_out/b32_c1.json 2>&1
timeout 900 python bench.py --config c3 --steps 2 --warmup 1 > gpurun_out/b32_c3.json 2>&1
timeout 900 python bench.py --config c4 --steps 2 --warmup 1 > gpurun_out/b32_c4.json 2>&1
timeout 900 python bench.py --config c4 --sampler dnc --chains 1 --steps 2 --warmup 1 > gpurun_out/b32_c4ref.json 2>&1
timeout 900 python bench.py --config c5 --steps 2 --warmup 1 > gpurun_out/b32_c5.json 2>&1
for f in gpurun_out/b32_*.json; do echo "== $f"; tail -c 400 $f; echo; done
