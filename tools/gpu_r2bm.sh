timeout 120 python tools/c4_kernels.py 1 3 | head -2
AUXMC_LIB_PATH=tools/_exp/ft512.so timeout 120 python tools/c4_kernels.py 1 3 | head -2
AUXMC_LIB_PATH=tools/_exp/ft256.so timeout 120 python tools/c4_kernels.py 1 3 | head -2
