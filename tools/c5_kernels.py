"""Per-kernel device times of one C5 aux-K iteration (spatio-temporal grid 4, d = 16,
T = 2^20, prefix backend + scan filter).  usage: c5_kernels.py [T] [iters]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2303_00301_b200 import _lib, auxk, bench_models as bm

T = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 20)
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
lib = _lib.load()
spec = bm.ModelSpec(kind="spatio-temporal", T=T, grid=4, data_seed=7)
lat, data = bm.simulate(spec)
tg = auxk.make_target(spec, data)
ch = auxk.init_chains(tg, lat, 5e-4, 1, 1)
ch.kernel_step(auxk.Backend.kPrefix, parallel_filter=True)
torch.cuda.synchronize()
lib.auxmc_profile_begin()
for _ in range(iters):
    ch.kernel_step(auxk.Backend.kPrefix, parallel_filter=True)
torch.cuda.synchronize()
tot, cnt = ctypes.c_double(0.0), ctypes.c_longlong(0)
names = ["k_pfg_elements", "k_pfg_elem_fill", "k_pfg_reduce_proto", "k_pfg_reduce_fill", "k_pfg_reduce<",
         "k_pfg_carry", "k_pfg_apply<", "k_pfg_apply_lanes", "k_pfg_recover<", "k_pfg_recover_lanes", "k_pfg_sum", "k_bwd_lean", "k_bwd_lanes", "k_pg_block_ops", "k_pg_block_offsets", "k_pg_carry", "k_pg_apply", "k_mma", "k_prefix",
         "k_path_terms", "k_gamma_terms", "k_build_aux", "k_grads", "k_aux"]
out = {}
for nm in names:
    lib.auxmc_profile_end(nm.encode(), ctypes.byref(tot), ctypes.byref(cnt)) if False else None
lib.auxmc_profile_end(b"", ctypes.byref(tot), ctypes.byref(cnt))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(iters):
    ch.kernel_step(auxk.Backend.kPrefix, parallel_filter=True)
e1.record()
torch.cuda.synchronize()
print(f"C5 T={T}: iteration {e0.elapsed_time(e1) / iters:.2f} ms (all kernels {tot.value / iters:.2f} ms)")
lib.auxmc_test_pfg_fixed_point_steps(1)
ch.kernel_step(auxk.Backend.kPrefix, parallel_filter=True)
torch.cuda.synchronize()
print(f"  vector-only scan-filter steps per iteration: {lib.auxmc_test_pfg_fixed_point_steps(1)}")
for nm in names:
    lib.auxmc_profile_begin()
    ch.kernel_step(auxk.Backend.kPrefix, parallel_filter=True)
    torch.cuda.synchronize()
    lib.auxmc_profile_end(nm.encode(), ctypes.byref(tot), ctypes.byref(cnt))
    print(f"  {nm:14s} {tot.value:8.3f} ms  ({cnt.value} launches)")
