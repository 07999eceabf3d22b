"""One C2 prefix-sampler workload for ncu capture (d=4, T=2^16, 1024 chains)."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2303_00301_b200 import lgssm, rng, bench_models as bm
mode = sys.argv[1] if len(sys.argv) > 1 else "pre"
sampler = int(sys.argv[2]) if len(sys.argv) > 2 else 1
T, B = 65536, 1024
spec = bm.ModelSpec(kind="lgssm-synthetic", T=T, dx=4, dy=1, data_seed=1)
lat, data = bm.simulate(spec)
m = bm.synthetic_lgssm(spec)
fr = lgssm.kalman_filter(m, data)
if mode == "pre":
    noise = lgssm.Noise.predrawn(torch.randn(B, 4, dtype=torch.float64, device="cuda"),
                                 torch.randn(B, T, 4, dtype=torch.float64, device="cuda"))
else:
    noise = lgssm.Noise.stream(rng.chain_keys(1, B))
ps = lgssm.PathSampler(m, B, sampler, True)
out = torch.empty(B, T + 1, 4, dtype=torch.float64, device="cuda")
for _ in range(3):
    ps(fr, noise, out)
torch.cuda.synchronize()
print("ok", float(out.abs().mean()))
