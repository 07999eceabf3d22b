mkdir -p gpurun_out
C3="python bench.py --config c3 --T 32 --chains 148 --steps 1 --warmup 1"
$C3 > gpurun_out/c3p.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_filter_seq|k_bwd_elements" -s 2 -c 2 -o gpurun_out/prof_c3_v2 $C3 > gpurun_out/ncu_c3.log 2>&1
tail -2 gpurun_out/ncu_c3.log
