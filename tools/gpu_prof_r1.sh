# Round-1 evidence: launch list of the bench command + one full capture of the top kernel.
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/r1_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1_launches.csv $CMD > gpurun_out/r1_ncu_launch.log 2>&1
$CMD > gpurun_out/r1_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_prefix_bulk -s 1 -c 1 -o gpurun_out/r1_prefix_full $CMD > gpurun_out/r1_ncu_full.log 2>&1
tail -2 gpurun_out/r1_ncu_launch.log gpurun_out/r1_ncu_full.log
