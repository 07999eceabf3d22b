mkdir -p gpurun_out
C3="python bench.py --config c3 --T 64 --steps 1 --warmup 1"
$C3 > gpurun_out/c3p.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_filter_seq -s 1 -c 1 -o gpurun_out/prof_c3_filter $C3 > gpurun_out/ncu_c3.log 2>&1
C4="python bench.py --config c4 --T 256 --chains 1 --steps 1 --warmup 1"
$C4 > gpurun_out/c4p.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_pit_forward -s 1 -c 1 -o gpurun_out/prof_c4_pit $C4 > gpurun_out/ncu_c4.log 2>&1
C1="python bench.py --config c1 --steps 2 --warmup 1"
$C1 > gpurun_out/c1p.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/c1_launches2.csv $C1 > /dev/null 2>&1
tail -2 gpurun_out/ncu_c3.log gpurun_out/ncu_c4.log
