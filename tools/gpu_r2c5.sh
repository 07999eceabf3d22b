timeout 300 python tools/c5_kernels.py 1048576 3 2>&1 | head -2
for v in lb64s2 lb64s4 lb128s2; do echo $v; AUXMC_LIB_PATH=tools/_exp/$v.so timeout 300 python tools/c5_kernels.py 1048576 3 2>&1 | head -1; done
