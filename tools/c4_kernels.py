"""Per-kernel device times of one C4 PIT iteration (stochvol d=3, N=256, T=2^14) for
C chains (default 1: the single-chain latency case).  usage: c4_kernels.py [C] [iters]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2303_00301_b200 import _lib, auxk, bench_models as bm, fkpg

C = int(sys.argv[1]) if len(sys.argv) > 1 else 1
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
lib = _lib.load()
T, N = 16384, 256
spec = bm.ModelSpec(kind="stochvol", T=T, dx=3, data_seed=11)
lat, data = bm.simulate(spec)
tg = auxk.make_target(spec, data)
ch = fkpg.init_pg(tg, torch.as_tensor(lat, device="cuda"), 1.0, 1, C, N)
ch.aux_pgibbs_step(fkpg.Variant.kPit)
torch.cuda.synchronize()
names = ["k_pit_forward_cluster", "k_pit_backward_table", "k_pit_backward_chase", "k_pit_particles",
         "k_pit_whiten", "k_pg_commit"]
res = {}
for nm in names:
    lib.auxmc_profile_begin()
    for _ in range(iters):
        ch.aux_pgibbs_step(fkpg.Variant.kPit)
    torch.cuda.synchronize()
    tot, cnt = ctypes.c_double(0.0), ctypes.c_longlong(0)
    lib.auxmc_profile_end(nm.encode(), ctypes.byref(tot), ctypes.byref(cnt))
    res[nm] = (tot.value / max(cnt.value, 1), cnt.value / iters)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(iters):
    ch.aux_pgibbs_step(fkpg.Variant.kPit)
e1.record()
torch.cuda.synchronize()
print(f"C4 PIT C={C}: iteration {e0.elapsed_time(e1) / iters:.2f} ms, status max {int(ch.status.max())}")
for nm, (ms, per) in res.items():
    print(f"  {nm:24s} {ms:8.3f} ms/launch x {per:.0f}")
