# Bit-identity check across two builds (a kernel change claimed not to alter results):
#   cp paper_2303_00301_b200/libauxmc_b200.so tools/_exp/old_lib.so   (before the change)
#   rebuild, then on the GPU box: bash tools/bitident.sh
#   AUXMC_LIB_PATH=<lib> python tools/_exp/bwd_bitident.py out.npz ; then compare npz files
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2303_00301_b200 import bench_models as bm, lgssm, rng, auxk
res = {}
for d, dy in ((5, 3), (16, 4), (40, 20), (64, 8)):
    spec = bm.ModelSpec(kind="lgssm-synthetic", T=120, dx=d, dy=dy, data_seed=3)
    lat, data = bm.simulate(spec)
    model = bm.synthetic_lgssm(spec)
    fr = lgssm.kalman_filter(model, data)
    keys = rng.chain_keys(7, 3)
    for smp in (0, 1, 2):
        try:
            x = lgssm.PathSampler(model, 3, smp, True)(fr, lgssm.Noise.stream(keys))
            res[f"d{d}_s{smp}"] = x.cpu().numpy()
        except Exception as e:
            print("skip", d, smp, e)
for name, spec, be, delta in (
        ("l96", bm.ModelSpec(kind="lorenz96", T=64, dx=40, data_seed=3), auxk.Backend.kSequential, 0.05),
        ("st", bm.ModelSpec(kind="spatio-temporal", T=512, grid=4, data_seed=7), auxk.Backend.kPrefix, 0.05)):
    lat, data = bm.simulate(spec)
    tg = auxk.make_target(spec, data)
    ch = auxk.init_chains(tg, lat, delta, 1, 4)
    for i in range(3):
        ch.kernel_step(be)
    res[name + "_x"] = ch.x.cpu().numpy()
    res[name + "_acc"] = ch.accepted.cpu().numpy()
from paper_2303_00301_b200 import fkpg
spec = bm.ModelSpec(kind="stochvol", T=256, dx=3, data_seed=11)
lat, data = bm.simulate(spec)
tg = auxk.make_target(spec, data)
for vname, var in (("pit", fkpg.Variant.kPit), ("ref", fkpg.Variant.kReference)):
    ch = fkpg.init_pg(tg, torch.as_tensor(lat, device="cuda"), 1.0, 1, 6, 256)
    for i in range(3):
        ch.aux_pgibbs_step(var)
    res["pg_" + vname + "_x"] = ch.x.cpu().numpy()
np.savez(sys.argv[1], **res)
print("saved", sorted(res))
