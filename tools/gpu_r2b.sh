# Round-2: the new bench line (headline C2 + every config record) and the reference arm.
mkdir -p gpurun_out/r2b
nproc > gpurun_out/r2b/host.txt; lscpu | head -20 >> gpurun_out/r2b/host.txt
( time timeout 900 python bench.py ) > gpurun_out/r2b/bench.json 2> gpurun_out/r2b/bench.err
( time timeout 900 python bench.py --impl reference ) > gpurun_out/r2b/bench_ref.json 2> gpurun_out/r2b/bench_ref.err
tail -c 3000 gpurun_out/r2b/bench.json; tail -5 gpurun_out/r2b/bench.err; cat gpurun_out/r2b/bench_ref.json
