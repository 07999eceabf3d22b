# Round-1 closing refresh after the DMMA edge-tile and DnC shared-bridge changes:
# GPU tests, smoke(), bench lines for every config, launch lists.
mkdir -p gpurun_out/r1f
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1f/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/r1f/pytest_gpu.log
tail -3 gpurun_out/r1f/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" > gpurun_out/r1f/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r1f/smoke.log
timeout 900 python bench.py > gpurun_out/r1f/r1f_bench_c2.json 2> gpurun_out/r1f/r1f_bench_c2.err
timeout 900 python bench.py --impl reference > gpurun_out/r1f/r1f_bench_ref.json 2> gpurun_out/r1f/r1f_bench_ref.err
for c in "--sampler dnc" "--config c1" "--config c3" "--config c4" "--config c5" "--config c5ts"; do
  n=$(echo $c | tr -d ' -')
  timeout 900 python bench.py $c --steps 3 --warmup 3 > gpurun_out/r1f/r1f_bench_$n.json 2> gpurun_out/r1f/r1f_bench_$n.err
done
C5="python bench.py --config c5 --steps 1 --warmup 1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r1f/r1f_c5_launches.csv $C5 > /dev/null 2>&1
ls -la gpurun_out/r1f
C3="python bench.py --config c3 --T 512 --steps 1 --warmup 1 --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r1f/r1f_c3_launches.csv $C3 > /dev/null 2>&1
C4="python bench.py --config c4 --T 2048 --steps 1 --warmup 1 --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r1f/r1f_c4_launches.csv $C4 > /dev/null 2>&1
C2="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r1f/r1f_c2_launches.csv $C2 > /dev/null 2>&1
ls gpurun_out/r1f
