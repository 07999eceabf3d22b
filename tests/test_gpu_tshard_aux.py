"""Time-sharded auxiliary Kalman step (tshard.ShardedAuxChain): one chain, the
horizon split over G ranks (threads on cuda:0 with an in-process exchange); each rank
works on its own time range only (the path is assembled from the ranks' ranges).
Every split must give the same bits (the super-block association of the
tshard scans does not depend on the rank count), and the chain must follow the
oracle's AuxChain with the prefix backend and the parallel filter
(auxk.cpp:130-198): identical accept decisions, paths to FP64 tolerance."""
import numpy as np
import pytest
import torch

from conftest import assert_close

pytestmark = pytest.mark.gpu

CASES = [
    ("spatio-temporal", dict(grid=3, data_seed=7), 150, 0.5),
    ("lgssm-synthetic", dict(dx=2, dy=1, data_seed=3), 300, 0.7),
    ("stochvol", dict(dx=3, data_seed=11), 120, 0.5),
    ("spatio-temporal", dict(grid=4, data_seed=7), 130, 0.01),  # d = 16 (C5)
]


@pytest.fixture(scope="module")
def mods():
    from paper_2303_00301_b200 import _lib, auxk, bench_models, tshard
    assert _lib.load().auxmc_device_ok() == 1
    return auxk, bench_models, tshard


def _run(mods, kind, kw, T, delta, world, steps, seed=4):
    auxk, bm, tshard = mods
    spec = bm.ModelSpec(kind=kind, T=T, **kw)
    lat, data = bm.simulate(spec)
    tg = auxk.make_target(spec, data)
    return tshard.LocalShardedAux.run(lambda: auxk.init_chains(tg, lat, delta, seed, 1),
                                      world, steps), lat, data


@pytest.mark.parametrize("kind,kw,T,delta", CASES)
def test_splits_bit_identical(mods, kind, kw, T, delta):
    ref, _, _ = _run(mods, kind, kw, T, delta, 1, 3)
    for world in (2, 3):
        got, _, _ = _run(mods, kind, kw, T, delta, world, 3)
        tshard = mods[2]
        assert torch.equal(tshard.LocalShardedAux.assemble(got), ref[0].x), f"G={world}: path"
        for ch in got:
            assert torch.equal(ch.log_gamma, ref[0].log_gamma)
            assert torch.equal(ch.accepted, ref[0].accepted)
            assert torch.equal(ch.iter, ref[0].iter)


@pytest.mark.parametrize("kind,kw,T,delta", CASES)
def test_matches_oracle(mods, oracle, kind, kw, T, delta):
    auxk, bm, tshard = mods
    steps, seed = 4, 4
    so = oracle.spec(kind, T=T, **kw)
    lat, data = oracle.simulate(so)
    otg = oracle.make_target(so, data)
    tg = auxk.make_target(bm.ModelSpec(kind=kind, T=T, **kw), data)
    ranks = [auxk.init_chains(tg, lat, delta, seed, 1) for _ in range(2)]
    o = oracle.AuxChain(otg, lat, delta)
    root = oracle.derive(oracle.from_seed(seed), oracle.L_CHAIN, 0)
    for it in range(steps):
        tshard.LocalShardedAux.run_on(ranks, 1)
        o.step(root, 1, 1)  # prefix backend, parallel filter
        assert int(ranks[0].accepted.cpu()[0]) == o.c.stats.accepted, f"step {it}"
    assert_close(tshard.LocalShardedAux.assemble(ranks)[0].cpu().numpy(), o.x, 1e-8, "path")
    assert_close(ranks[0].log_gamma[0].cpu(), o.c.log_gamma, 1e-8, "log_gamma")


def test_exchange_is_aggregates_not_paths(mods):
    """per step the ranks exchange super-block aggregates, the
    sampler's block rows, 2 d halo doubles and the step's super-block partials — no
    path-length tensor (the round-1 step all-gathered the whole proposal)."""
    auxk, bm, tshard = mods
    T = 3000
    spec = bm.ModelSpec(kind="spatio-temporal", T=T, grid=3, data_seed=7)
    lat, data = bm.simulate(spec)
    tg = auxk.make_target(spec, data)
    sizes = []
    orig = tshard.ShardedAuxChain.step

    def traced(self):
        ex = self.exchange

        def rec(t):
            sizes.append(t.numel())
            return ex(t)
        self.exchange = rec
        try:
            orig(self)
        finally:
            self.exchange = ex
    tshard.ShardedAuxChain.step = traced
    try:
        tshard.LocalShardedAux.run(lambda: auxk.init_chains(tg, lat, 0.5, 4, 1), 2, 1)
    finally:
        tshard.ShardedAuxChain.step = orig
    d = 9
    assert max(sizes) < (T + 1) * d // 4, sizes
