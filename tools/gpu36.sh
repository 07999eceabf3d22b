C1="python bench.py --config c1 --steps 3 --warmup 1 --no-graph"
$C1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/c1_launches.csv $C1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/c1_launches.csv | head -40
