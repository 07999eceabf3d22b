# Round-1 final evidence: bench lines for every config + launch lists of the
# configs changed since r1b (C1, C5, C5 time-sharded).
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r1c_bench_c2.json 2> gpurun_out/r1c_bench_c2.err
timeout 900 python bench.py --impl reference > gpurun_out/r1c_bench_ref.json 2> gpurun_out/r1c_bench_ref.err
for c in "--sampler dnc" "--config c1" "--config c3" "--config c4" "--config c5" "--config c5ts"; do
  n=$(echo $c | tr -d ' -')
  timeout 900 python bench.py $c --steps 3 --warmup 3 > gpurun_out/r1c_bench_$n.json 2> gpurun_out/r1c_bench_$n.err
done
C1="python bench.py --config c1 --steps 2 --warmup 1 --no-graph"
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r1c_c1_launches.csv $C1 > /dev/null 2>&1
C5="python bench.py --config c5 --steps 1 --warmup 1"
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r1c_c5_launches.csv $C5 > /dev/null 2>&1
ls -la gpurun_out/r1c_*
