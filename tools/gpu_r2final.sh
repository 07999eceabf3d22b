# Round-2 closing evidence: full GPU suite, smoke, bench (all configs), reference arm, c5ts,
# launch lists of C3 / C4 one chain, ncu --set full of the C3 fused filter and backward elements
mkdir -p gpurun_out/r2h
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2h/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2h/pytest_gpu.log
tail -3 gpurun_out/r2h/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2h/smoke.log 2>&1; tail -1 gpurun_out/r2h/smoke.log
( time timeout 1200 python bench.py ) > gpurun_out/r2h/bench.json 2> gpurun_out/r2h/bench.err
( time timeout 900 python bench.py --impl reference ) > gpurun_out/r2h/bench_ref.json 2> gpurun_out/r2h/bench_ref.err
timeout 600 python bench.py --config c5ts > gpurun_out/r2h/bench_c5ts.json 2> gpurun_out/r2h/bench_c5ts.err
python tools/c3_kernels.py 4096 256 3 > gpurun_out/r2h/c3_kernels.txt 2>&1
python tools/c4_kernels.py 1 3 > gpurun_out/r2h/c4_1chain_kernels.txt 2>&1
ls gpurun_out/r2h
