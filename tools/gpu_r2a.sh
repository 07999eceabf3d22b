# Round-2 opening check: GPU tests, smoke, default bench line.
mkdir -p gpurun_out/r2a
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2a/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/r2a/pytest_gpu.log
tail -3 gpurun_out/r2a/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" > gpurun_out/r2a/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2a/smoke.log
timeout 600 python bench.py > gpurun_out/r2a/bench_c2.json 2> gpurun_out/r2a/bench_c2.err
nproc > gpurun_out/r2a/host.txt; lscpu | head -20 >> gpurun_out/r2a/host.txt
cat gpurun_out/r2a/bench_c2.json
