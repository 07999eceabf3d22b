mkdir -p gpurun_out/r2ai
python tools/c3_kernels.py 4096 256 3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bwd_lean -c 1 -o gpurun_out/r2ai/bwd_full python bench.py --config c3 --T 256 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r2ai/ncu.log 2>&1
