mkdir -p gpurun_out/r2y3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2y3/c3_launches.csv python bench.py --config c3 --T 512 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2y3/c3_launches.csv > gpurun_out/r2y3/c3_launches.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_filter_direct -c 1 -o gpurun_out/r2y3/fd_full python bench.py --config c3 --T 256 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bwd_lean -c 1 -o gpurun_out/r2y3/bwd_full python bench.py --config c3 --T 256 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2y3/c4_1chain_launches.csv python bench.py --config c4 --chains 1 --variant pit --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2y3/c4_1chain_launches.csv > gpurun_out/r2y3/c4_1chain_launches.txt 2>&1
ls gpurun_out/r2y3
