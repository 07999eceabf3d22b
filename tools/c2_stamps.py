"""Per-phase clock64 stamps of the C2 kernel (prefix_mma.cu built with -DAUXMC_PM_EXP=9: tools/exp_build.sh m9 prefix_mma.cu -DAUXMC_PM_EXP=9)."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_2303_00301_b200 import lgssm, rng, bench_models as bm
T, B = 65536, 1024
spec = bm.ModelSpec(kind="lgssm-synthetic", T=T, dx=4, dy=1, data_seed=1)
lat, data = bm.simulate(spec)
m = bm.synthetic_lgssm(spec)
fr = lgssm.kalman_filter(m, data)
keys = rng.chain_keys(1, B)
noise = lgssm.Noise.predrawn(rng.normals(keys, rng.kTerminalDraw, 0, 1, 4).reshape(B, 4),
                             rng.normals(keys, rng.kBackwardNoise, 0, T, 4))
ps = lgssm.PathSampler(m, B, 1, True)
out = torch.empty(B, T + 1, 4, dtype=torch.float64, device="cuda")
for _ in range(3):
    ps(fr, noise, out)
torch.cuda.synchronize()
ts = out[0].flatten()[:128].view(torch.int64).cpu().numpy().reshape(16, 8)
names = ["cw_top", "cw_issued", "cw_tile", "cw_B_done", "c0_top", "c0_A_done", "c0_bar1", "c0_C_done"]
base = ts[0, 0]
print("iter " + " ".join(f"{n:>10s}" for n in names))
for i in range(16):
    print(f"{i:4d} " + " ".join(f"{int(v - base):10d}" for v in ts[i]))
d = ts[1:, 0] - ts[:-1, 0]
print("cycles per superchunk (cw_top deltas):", d.mean())
print("mean: issue", (ts[:, 1] - ts[:, 0]).mean(), "tile wait", (ts[:, 2] - ts[:, 1]).mean(),
      "phase B", (ts[:, 3] - ts[:, 2]).mean(), "| A", (ts[:, 5] - ts[:, 4]).mean(),
      "bar1 wait(c0)", (ts[:, 6] - ts[:, 5]).mean(), "C", (ts[:, 7] - ts[:, 6]).mean(),
      "bar2->next", (ts[1:, 4] - ts[:-1, 7]).mean())
