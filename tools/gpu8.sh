mkdir -p gpurun_out
C3="python bench.py --config c3 --T 256 --steps 1 --warmup 1"
$C3 > gpurun_out/c3_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/c3_launches.csv $C3 > /dev/null 2>&1
C4="python bench.py --config c4 --T 1024 --chains 1 --steps 1 --warmup 1"
$C4 > gpurun_out/c4_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/c4_launches.csv $C4 > /dev/null 2>&1
C1="python bench.py --config c1 --steps 2 --warmup 1"
$C1 > gpurun_out/c1_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/c1_launches.csv $C1 > /dev/null 2>&1
ls -la gpurun_out/*launches.csv
