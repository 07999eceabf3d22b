"""Quick C2 timing (prefix / seq / dnc samplers, d=4, T=2^16, 1024 chains)."""
import sys, time, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2303_00301_b200 import lgssm, rng, _lib, pit

T = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
from paper_2303_00301_b200 import bench_models as bm
spec = bm.ModelSpec(kind="lgssm-synthetic", T=T, dx=4, dy=1, data_seed=1)
lat, data = bm.simulate(spec)
m = bm.synthetic_lgssm(spec)
t0 = time.time(); fr = lgssm.kalman_filter(m, data); torch.cuda.synchronize()
print("filter s", time.time() - t0, "status", int(fr.status[0]), "ll", float(fr.log_marginal[0]))
keys = rng.chain_keys(1, B)
g = np.random.default_rng(0)
term = torch.randn(B, 4, dtype=torch.float64, device="cuda")
back = torch.randn(B, T, 4, dtype=torch.float64, device="cuda")
for name, sampler, noise in [("prefix-pre", 1, lgssm.Noise.predrawn(term, back)),
                             ("prefix-rng", 1, lgssm.Noise.stream(keys)),
                             ("seq-pre", 0, lgssm.Noise.predrawn(term, back)),
                             ("seq-rng", 0, lgssm.Noise.stream(keys)),
                             ("dnc-rng", 2, lgssm.Noise.stream(keys))]:
    ps = lgssm.PathSampler(m, B, sampler, True)
    out = torch.empty(B, T + 1, 4, dtype=torch.float64, device="cuda")
    for _ in range(3): ps(fr, noise, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    e0.record()
    for _ in range(n): ps(fr, noise, out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    ct = B * (T + 1)
    bytes_ = ct * (64 if "pre" in name else 32)
    print(f"{name:12s} {ms:8.3f} ms  {ct/ms/1e6:8.2f} Gct/s  {bytes_/ms/1e6:8.1f} GB/s  status={int(ps.status.max())}")
