"""Time-sharded scan filter: pit::parallel_filter split over
ranks by super-blocks with one all-gather of aggregates.  Every split reproduces
the one-rank result bit for bit; results match the oracle's filter."""
import json
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

from conftest import ROOT, assert_close
from testutil import random_model, simulate_obs, to_gpu_model

pytestmark = pytest.mark.gpu


def _assemble(tshard, frs, shards, T):
    fm = torch.empty_like(frs[0].filt_mean)
    fc = torch.empty_like(frs[0].filt_cov)
    pm = torch.empty_like(frs[0].pred_mean)
    pc = torch.empty_like(frs[0].pred_cov)
    for fr, sh in zip(frs, shards):
        sl = slice(sh.t_lo, sh.t_hi)
        fm[:, sl], fc[:, sl], pm[:, sl], pc[:, sl] = (fr.filt_mean[:, sl], fr.filt_cov[:, sl],
                                                      fr.pred_mean[:, sl], fr.pred_cov[:, sl])
    return fm, fc, pm, pc


@pytest.mark.parametrize("T,dx,dy,seed", [(3000, 3, 2, 61), (700, 10, 4, 62), (4500, 2, 1, 63)])
def test_tshard_filter_bit_identical_for_every_split(oracle, T, dx, dy, seed):
    from paper_2303_00301_b200 import tshard
    s = oracle.derive(oracle.from_seed(seed), oracle.L_SIMULATE, 2)
    m = random_model(s, T, dx, dy, True, True)
    obs = simulate_obs(m, oracle.from_seed(seed + 100))
    gm = to_gpu_model(m)
    g = tshard.TShardGeom.of(T, dx)
    assert g.nsup >= 3, g
    base = None
    for world in (1, 2, 3, min(8, g.nsup)):
        shards, frs, lm = tshard.LocalExchange.run(gm, obs, world)
        got = _assemble(tshard, frs, shards, T) + (lm,)
        for sh in shards:
            assert int(sh.status[0]) == 0
        if base is None:
            base = got
            want = oracle.kalman_filter(m, obs)
            assert_close(got[0][0].cpu(), want.filt_mean, 1e-8, "filt_mean")
            assert_close(got[1][0].cpu(), want.filt_cov, 1e-8, "filt_cov")
            assert_close(got[2][0].cpu(), want.pred_mean, 1e-8, "pred_mean")
            assert_close(got[3][0].cpu(), want.pred_cov, 1e-8, "pred_cov")
            assert_close(lm.cpu(), [want.log_marginal], 1e-9, "log_marginal")
        else:
            for a, b in zip(got, base):
                assert torch.equal(a, b), f"world {world} differs from world 1"


def test_tshard_world2_gloo_processes(tmp_path):
    """Two processes, gloo all-gather, both driving cuda:0: bit-identical to one rank."""
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    out = tmp_path / "tshard.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           str(ROOT / "tests" / "mp" / "tshard_worker.py"), str(out)]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.load(open(out))
    assert res["world"] == 2 and res["bit_identical"], res
    assert res["lm_rel_err"] < 1e-9, res
    assert res["aux_bit_identical"], res


@pytest.mark.parametrize("T,dx,dy,seed", [(3000, 3, 2, 81), (1200, 10, 4, 82)])
def test_tshard_prefix_bit_identical_and_matches_oracle(oracle, T, dx, dy, seed):
    """Sharded prefix sampler: every split gives the same path bits; the path is the
    oracle's prefix_sample (stream noise, same key) to FP64 tolerance."""
    from paper_2303_00301_b200 import lgssm, rng, tshard
    s = oracle.derive(oracle.from_seed(seed), oracle.L_SIMULATE, 2)
    m = random_model(s, T, dx, dy, True, False)
    obs = simulate_obs(m, oracle.from_seed(seed + 100))
    gm = to_gpu_model(m)
    keys = rng.chain_keys(seed, 1)
    noise = lgssm.Noise.stream(keys)
    g = tshard.TShardGeom.of(T, dx)
    base = None
    for world in (1, 2, 3, min(8, g.nsup)):
        shards, frs, lm, trajs = tshard.LocalExchange.run(gm, obs, world, noise)
        path = torch.empty_like(trajs[0])
        for sh, tr in zip(shards, trajs):
            path[sh.t_lo:min(sh.t_hi, T)] = tr[sh.t_lo:min(sh.t_hi, T)]
        path[T] = trajs[-1][T]
        for tr in trajs:
            assert torch.equal(tr[T], path[T])
        if base is None:
            base = path
            fr_o = oracle.kalman_filter(m, obs)
            want = oracle.prefix_sample(m, fr_o, oracle.stream_noise(
                oracle.derive(oracle.from_seed(seed), oracle.L_CHAIN, 0)))
            assert_close(path.cpu(), want, 1e-8, "sharded prefix path")
        else:
            assert torch.equal(path, base), f"world {world} path differs"
