"""One rank of the time-sharded scan filter test (tests/test_gpu_tshard.py):
launched by torch.distributed.run with the gloo backend; every rank drives its
own time range on cuda:0 (no kernel waits on another rank: the exchange is a
host all-gather), rank 0 compares with a one-rank run and writes a verdict."""
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main(out_path):
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    from oracle import pyoracle as O
    from testutil import random_model, simulate_obs, to_gpu_model
    from paper_2303_00301_b200 import tshard
    s = O.derive(O.from_seed(71), O.L_SIMULATE, 2)
    m = random_model(s, 2500, 3, 2, True, True)
    obs = simulate_obs(m, O.from_seed(72))
    gm = to_gpu_model(m)
    from paper_2303_00301_b200 import lgssm, rng
    noise = lgssm.Noise.stream(rng.chain_keys(73, 1))
    fr, lm, traj, (t_lo, t_hi) = tshard.sharded_filter_and_prefix(gm, obs, noise, rank, world,
                                                                   tshard.torch_exchange())
    torch.cuda.synchronize()
    sl = slice(t_lo, t_hi)
    ps = slice(t_lo, min(t_hi, m.T))
    mine = torch.cat([fr.filt_mean[0, sl].reshape(-1), fr.filt_cov[0, sl].reshape(-1),
                      fr.pred_mean[0, sl].reshape(-1), fr.pred_cov[0, sl].reshape(-1),
                      traj[ps].reshape(-1), traj[m.T]]).cpu()
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([mine.numel()]))
    nmax = int(max(int(n) for n in sizes))
    padded = torch.zeros(nmax, dtype=torch.float64)
    padded[:mine.numel()] = mine
    parts = [torch.zeros(nmax, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, padded)
    parts = [p[:int(n)] for p, n in zip(parts, sizes)]
    if rank == 0:
        shards, frs, lm1, trajs = tshard.LocalExchange.run(gm, obs, 1, noise)
        ref, rtraj = frs[0], trajs[0]
        ok = True
        for r in range(world):
            g = tshard.TShardGeom.of(m.T, m.dx)
            _, _, a, b = g.owned(r, world)
            want = torch.cat([ref.filt_mean[0, a:b].reshape(-1), ref.filt_cov[0, a:b].reshape(-1),
                              ref.pred_mean[0, a:b].reshape(-1),
                              ref.pred_cov[0, a:b].reshape(-1),
                              rtraj[a:min(b, m.T)].reshape(-1), rtraj[m.T]]).cpu()
            ok = ok and torch.equal(parts[r], want)
        ok = ok and torch.equal(lm.cpu(), lm1.cpu())
        want_o = O.kalman_filter(m, obs)
        err = abs(float(lm1.item()) - want_o.log_marginal) / max(1.0, abs(want_o.log_marginal))
        res = {"bit_identical": bool(ok), "world": world, "lm_rel_err": err}
    # the full auxiliary Kalman step, time-sharded over the ranks
    from paper_2303_00301_b200 import auxk, bench_models as bm
    spec = bm.ModelSpec(kind="spatio-temporal", T=300, grid=3, data_seed=7)
    lat, data = bm.simulate(spec)
    tg = auxk.make_target(spec, data)
    ch = auxk.init_chains(tg, lat, 0.5, 9, 1)
    sa = tshard.ShardedAuxChain(ch, rank, world, tshard.torch_exchange())
    for _ in range(3):
        sa.step()
    torch.cuda.synchronize()
    if rank == 0:
        one = tshard.LocalShardedAux.run(lambda: auxk.init_chains(tg, lat, 0.5, 9, 1), 1, 3)[0]
        lo, hi = sa.t_lo, sa.t_hi  # this rank's own rows (plus the right halo row)
        res["aux_bit_identical"] = bool(torch.equal(one.x[:, lo:hi + 1], ch.x[:, lo:hi + 1]) and
                                        torch.equal(one.log_gamma, ch.log_gamma) and
                                        torch.equal(one.accepted, ch.accepted))
        res["aux_accepted"] = int(ch.accepted.cpu()[0])
        json.dump(res, open(out_path, "w"))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
