mkdir -p gpurun_out/r2ba
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2ba/c2_launches.csv python bench.py --config c2 --steps 3 --warmup 3 --no-e2e --no-cpu --no-check > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2ba/c2_launches.csv | head
