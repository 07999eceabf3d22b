timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file gpurun_out/r2m_c4_1chain_launches.csv python bench.py --config c4 --chains 1 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2m_c4_1chain_launches.csv | head -12
