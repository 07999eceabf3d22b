timeout 300 python tools/c3_kernels.py 4096 256 3 | grep -E "step|seq"
AUXMC_LIB_PATH=tools/_exp/sq200.so timeout 300 python tools/c3_kernels.py 4096 256 3 | grep -E "step|seq"
AUXMC_LIB_PATH=tools/_exp/sq80.so timeout 300 python tools/c3_kernels.py 4096 256 3 | grep -E "step|seq"
