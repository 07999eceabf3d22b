# Round-2 mid-session evidence: full GPU suite, smoke, full bench (all configs), reference arm,
# c5ts, launch lists for C2 / C4 one chain / C5ts, ncu of the C2 kernel with clock-control none
mkdir -p gpurun_out/r2t
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2t/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2t/pytest_gpu.log
tail -3 gpurun_out/r2t/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2t/smoke.log 2>&1; tail -1 gpurun_out/r2t/smoke.log
( time timeout 900 python bench.py ) > gpurun_out/r2t/bench.json 2> gpurun_out/r2t/bench.err
( time timeout 900 python bench.py --impl reference ) > gpurun_out/r2t/bench_ref.json 2> gpurun_out/r2t/bench_ref.err
timeout 600 python bench.py --config c5ts > gpurun_out/r2t/bench_c5ts.json 2> gpurun_out/r2t/bench_c5ts.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2t/c5ts_launches.csv python bench.py --config c5ts --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2t/c3_launches.csv python bench.py --config c3 --T 512 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_prefix_mma -c 1 -o gpurun_out/r2t/c2_mma_full python bench.py --config c2 --steps 1 --warmup 1 --no-e2e --no-cpu --no-check > /dev/null 2>&1
ls gpurun_out/r2t
