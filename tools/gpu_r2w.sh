mkdir -p gpurun_out/r2w
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_filter_direct -c 1 -o gpurun_out/r2w/fd_full python bench.py --config c3 --T 256 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r2w/ncu.log 2>&1
tail -3 gpurun_out/r2w/ncu.log
ls gpurun_out/r2w
