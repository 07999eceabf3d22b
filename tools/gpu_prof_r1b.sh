# Round-1 evidence refresh: launch lists (C2 bench command, C3, C5) + full capture of the C2 top kernel.
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/r1b_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1b_c2_launches.csv $CMD > gpurun_out/r1b_ncu_launch.log 2>&1
$CMD > gpurun_out/r1b_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_prefix_bulk -s 1 -c 1 -o gpurun_out/r1b_prefix_full $CMD > gpurun_out/r1b_ncu_full.log 2>&1
C3="python bench.py --config c3 --T 512 --steps 1 --warmup 1"
$C3 > gpurun_out/r1b_c3_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r1b_c3_launches.csv $C3 > /dev/null 2>&1
C5="python bench.py --config c5 --steps 1 --warmup 1"
$C5 > gpurun_out/r1b_c5_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r1b_c5_launches.csv $C5 > /dev/null 2>&1
C4="python bench.py --config c4 --steps 1 --warmup 1"
$C4 > gpurun_out/r1b_c4_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r1b_c4_launches.csv $C4 > /dev/null 2>&1
ls -la gpurun_out/r1b_*
