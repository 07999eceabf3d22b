python tools/c5_kernels.py
AUXMC_LIB_PATH=tools/_exp/bl16.so python tools/c5_kernels.py
