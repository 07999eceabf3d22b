# Round-1 final refresh: GPU tests, then bench lines for every config and the C5
# launch list (after the bwd-element, blocked-LLT and cSMC running-sum changes).
mkdir -p gpurun_out/r1e
timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/r1e/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/r1e/pytest_gpu.log
tail -3 gpurun_out/r1e/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r1e/r1e_bench_c2.json 2> gpurun_out/r1e/r1e_bench_c2.err
timeout 900 python bench.py --impl reference > gpurun_out/r1e/r1e_bench_ref.json 2> gpurun_out/r1e/r1e_bench_ref.err
for c in "--sampler dnc" "--config c1" "--config c3" "--config c4" "--config c5" "--config c5ts"; do
  n=$(echo $c | tr -d ' -')
  timeout 900 python bench.py $c --steps 3 --warmup 3 > gpurun_out/r1e/r1e_bench_$n.json 2> gpurun_out/r1e/r1e_bench_$n.err
done
C5="python bench.py --config c5 --steps 1 --warmup 1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r1e/r1e_c5_launches.csv $C5 > /dev/null 2>&1
ls -la gpurun_out/r1e
C3="python bench.py --config c3 --T 512 --steps 1 --warmup 1 --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r1e/r1e_c3_launches.csv $C3 > /dev/null 2>&1
C4="python bench.py --config c4 --T 2048 --steps 1 --warmup 1 --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r1e/r1e_c4_launches.csv $C4 > /dev/null 2>&1
C2="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r1e/r1e_c2_launches.csv $C2 > /dev/null 2>&1
ls gpurun_out/r1e
