mkdir -p gpurun_out
A="bench.py --steps 2 --warmup 1 --no-e2e --no-cpu"
SKIP=1 bash tools/prof.sh k_prefix_bulk prof_c2_pfx $A
