"""clock64 phase stamps of one C3 backward-elements item (k_bwd_lean built with
-DAUXMC_BWD_EXP=9: tools/exp_build.sh bwst sample.cu -DAUXMC_BWD_EXP=9)."""
import ctypes
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2303_00301_b200 import _lib, auxk, bench_models as bm

lib = _lib.load()
spec = bm.ModelSpec(kind="lorenz96", T=512, dx=40, data_seed=3)
lat, data = bm.simulate(spec)
tg = auxk.make_target(spec, data)
ch = auxk.init_chains(tg, lat, 0.05, 1, 256)
ch.kernel_step(0)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * 64)()
lib.auxmc_debug_bwd_stamps(buf, 64)
s = np.array(buf[:11], dtype=np.int64)
names = ["load+C", "zero-check", "chol S", "trsm L", "Lambda dmma", "trsm L^T", "mirror/off", "-",
         "chol Lambda", "write"]
d = np.diff(s)
print("item total", s[10] - s[0])
for n, v in zip(names, d):
    print(f"  {n:12s} {v}")
