"""Per-phase clock64 stamps of one filter step (t = 200, CTA 0) of the fused direct
filter (filter_direct.cu built with -DAUXMC_FD_EXP=9: tools/exp_build.sh fdst
filter_direct.cu -DAUXMC_FD_EXP=9; run with AUXMC_LIB_PATH=tools/_exp/fdst.so)."""
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
for _ in range(2):
    ch.kernel_step(0)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * 4096)()
lib.auxmc_debug_fd_stamps(buf, 4096)
st = np.array(buf[:], dtype=np.int64).reshape(8, 512)
w0 = st[0]
base = w0[0]
print("warp0: predict+obs", w0[1] - w0[0], "covs write", w0[2] - w0[1])
pan = []
for p in range(10):
    a, b, c = w0[8 + 3 * p], w0[9 + 3 * p], w0[10 + 3 * p]
    prev = w0[2] if p == 0 else w0[10 + 3 * (p - 1)]
    pan.append((a - prev, b - a, c - b))
pan = np.array(pan)
print("per panel (mean over 10): to-barrierA %.0f  dinv+barrierB %.0f  dmma %.0f" % tuple(pan.mean(0)))
print("panels:", pan.tolist())
print("fill (first panel to-barrierA)", pan[0, 0])
print("after elim -> sync", w0[41] - w0[40], "tail", w0[42] - w0[41], "elim total", w0[40] - w0[2])
print("step total", w0[42] - w0[0])
for wi in range(1, 8):
    print(f"warp{wi}: dmma per panel", np.mean([st[wi][10 + 3 * p] - st[wi][9 + 3 * p] for p in range(10)]))
