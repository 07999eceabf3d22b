C="python bench.py --sampler dnc --no-cpu --no-e2e --steps 2 --warmup 1"
$C > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/dnc_launches.csv $C > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/dnc_launches.csv | head -14
