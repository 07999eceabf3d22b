mkdir -p gpurun_out
A="bench.py --config c3 --T 16 --chains 148 --steps 1 --warmup 1"
bash tools/prof.sh k_filter_seq prof_c3_filt3 $A
bash tools/prof.sh k_bwd_elements prof_c3_bwd3 $A
