# Round-2 closing evidence: full GPU suite, smoke, bench (all configs), reference arm, c5ts,
# launch lists of C3 / C4 one chain, ncu --set full of the C3 fused filter and backward elements
mkdir -p gpurun_out/r2k
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2k/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2k/pytest_gpu.log
tail -3 gpurun_out/r2k/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2k/smoke.log 2>&1; tail -1 gpurun_out/r2k/smoke.log
( time timeout 1200 python bench.py ) > gpurun_out/r2k/bench.json 2> gpurun_out/r2k/bench.err
( time timeout 900 python bench.py --impl reference ) > gpurun_out/r2k/bench_ref.json 2> gpurun_out/r2k/bench_ref.err
timeout 600 python bench.py --config c5ts > gpurun_out/r2k/bench_c5ts.json 2> gpurun_out/r2k/bench_c5ts.err
python tools/c3_kernels.py 4096 256 3 > gpurun_out/r2k/c3_kernels.txt 2>&1
python tools/c4_kernels.py 1 3 > gpurun_out/r2k/c4_1chain_kernels.txt 2>&1
ls gpurun_out/r2k
python tools/c5_kernels.py 1048576 3 > gpurun_out/r2k/c5_kernels.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2k/c5_launches.csv python bench.py --config c5 --steps 1 --warmup 1 > gpurun_out/r2k/c5_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_pfg_apply_lanes|k_pfg_reduce_fill|k_pfg_reduce_proto4" -s 3 -c 3 -o gpurun_out/r2k/c5_full python tools/c5_kernels.py 65536 1 > gpurun_out/r2k/c5_full.log 2>&1
ncu -i gpurun_out/r2k/c5_full.ncu-rep --page raw --csv > gpurun_out/r2k/c5_full_raw.csv 2>&1
rm -f gpurun_out/r2k/c5_full.ncu-rep
ls -la gpurun_out/r2k
