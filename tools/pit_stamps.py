"""clock64 stamps of the cluster PIT forward pass (csmc.cu with -DAUXMC_PIT_EXP=9:
tools/exp_build.sh p9 csmc.cu -DAUXMC_PIT_EXP=9), C4 1 chain; timing only."""
import sys, pathlib
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2303_00301_b200 import auxk, bench_models as bm, fkpg, _lib
spec = bm.ModelSpec(kind="stochvol", T=16384, dx=3, data_seed=11)
lat, data = bm.simulate(spec)
tg = auxk.make_target(spec, data)
ch = fkpg.init_pg(tg, lat, 1.0, 1, 1, 256)
lib = _lib.load()
n = lib.auxmc_aux_pgibbs_workspace(ch.target.raw(), 1, 256, 1)
ch.aux_pgibbs_step(fkpg.Variant.kPit)
torch.cuda.synchronize()
# the stamps overwrite the first 128 doubles of the workspace's forward-message block
import ctypes
ws = ch._ws
# locate a.Wt: after it (C), u, mq, part in the arena (256-B aligned takes)
def al(x): return (x + 255) // 256 * 256
T, N, d = 16384, 256, 3
off = al(8) + al(8 * (T + 1) * d) * 2 + al(8 * (T + 1) * N * d)
ts = ws[off:off + 128 * 8].cpu().numpy().view(np.int64).reshape(16, 8)
names = ["top", "am+ai", "pairs", "combine+push", "cluster_sync"]
d = ts[:, 1:5] - ts[:, 0:4]
print("per-phase cycles (mean over 16 steps):", dict(zip(names[1:], d.mean(0).round(0))))
print("per step:", (ts[1:, 0] - ts[:-1, 0]).mean())
