mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/b28_c2.json 2> gpurun_out/b28_c2.err; tail -c 3000 gpurun_out/b28_c2.json
timeout 600 python bench.py --config c1 --steps 20 --warmup 5 > gpurun_out/b28_c1.json 2>&1; tail -c 600 gpurun_out/b28_c1.json
timeout 900 python bench.py --config c3 --steps 2 --warmup 1 > gpurun_out/b28_c3.json 2>&1; tail -c 600 gpurun_out/b28_c3.json
timeout 900 python bench.py --config c4 --steps 2 --warmup 1 > gpurun_out/b28_c4.json 2>&1; tail -c 600 gpurun_out/b28_c4.json
timeout 900 python bench.py --config c5 --steps 2 --warmup 1 > gpurun_out/b28_c5.json 2>&1; tail -c 600 gpurun_out/b28_c5.json
