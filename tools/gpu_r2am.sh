python tools/c3_kernels.py 4096 256 3 | head -2
AUXMC_LIB_PATH=tools/_exp/fdbf.so python tools/c3_kernels.py 4096 256 3 | head -2
AUXMC_LIB_PATH=tools/_exp/fdbfst.so python tools/fd_stamps.py
