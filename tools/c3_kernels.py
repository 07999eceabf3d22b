"""Per-kernel device times of the C3 aux step (CUDA events around each launch of the
named kernels, auxmc_profile_*), for A/B work on the structure-aware path.

usage: python tools/c3_kernels.py [T] [C] [iters]"""
import ctypes
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))

from paper_2303_00301_b200 import _lib, auxk, bench_models as bm

T = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
C = int(sys.argv[2]) if len(sys.argv) > 2 else 256
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
lib = _lib.load()
spec = bm.ModelSpec(kind="lorenz96", T=T, dx=40, data_seed=3)
lat, data = bm.simulate(spec)
tg = auxk.make_target(spec, data)
ch = auxk.init_chains(tg, lat, 0.05, 1, C)
ch.kernel_step(0)
torch.cuda.synchronize()
names = ["k_filter_direct", "k_bwd_lean", "k_seq_sample", "k_path_terms", "k_build_aux",
         "k_gamma_terms"]
res = {}
for nm in names:
    lib.auxmc_profile_begin()
    for _ in range(iters):
        ch.kernel_step(0)
    torch.cuda.synchronize()
    tot, cnt = ctypes.c_double(0.0), ctypes.c_longlong(0)
    lib.auxmc_profile_end(nm.encode(), ctypes.byref(tot), ctypes.byref(cnt))
    res[nm] = (tot.value / max(cnt.value, 1), cnt.value / iters)
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
for _ in range(iters):
    ch.kernel_step(0)
ev1.record()
torch.cuda.synchronize()
print(f"T={T} C={C}: step {ev0.elapsed_time(ev1) / iters:.2f} ms")
for nm, (ms, per) in res.items():
    print(f"  {nm:18s} {ms:8.3f} ms/launch x {per:.0f} per step")
