mkdir -p gpurun_out
AUXMC_LIB_PATH=$PWD/${OLD_LIB:-tools/_exp/old_lib.so} timeout 300 python tools/bitident.py gpurun_out/old.npz
timeout 300 python tools/bitident.py gpurun_out/new.npz
python - <<'PY'
import numpy as np
a=np.load("gpurun_out/old.npz"); b=np.load("gpurun_out/new.npz")
for k in sorted(a):
    print(k, a[k].shape, "BIT-IDENTICAL" if a[k].tobytes()==b[k].tobytes() else "DIFF %g" % np.max(np.abs(a[k]-b[k])))
PY
