mkdir -p gpurun_out
python tools/prof_prefix.py pre 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_prefix_shared -s 2 -c 1 -o gpurun_out/prof_prefix_v1 python tools/prof_prefix.py pre 1 > gpurun_out/ncu.log 2>&1
tail -5 gpurun_out/ncu.log
