python tools/c3_kernels.py 4096 256 3
AUXMC_LIB_PATH=tools/_exp/bw5.so python tools/c3_kernels.py 4096 256 3 | head -3
