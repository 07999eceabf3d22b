A="bench.py --config c3 --T 32 --chains 148 --steps 1 --warmup 1"
SKIP=1 bash tools/prof.sh k_bwd_elements prof_c3_bwd8 $A
