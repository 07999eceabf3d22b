"""GPU parity of the auxiliary Kalman MH kernel against the oracle.

Same targets, same chain roots (from_seed(seed).derive(kChain, c)), same
iteration streams: per-step accept/reject decisions must agree exactly and
paths, log γ and log α to FP64 tolerance.  Mirrors
proj/tests/test_target_auxk.cpp: exact targets accept every move with
|log α| ~ 0 (:182-231), generic potentials give a proper MH step, all three
backends share decisions (:292-315), δ adaptation (:334-372).
"""
import numpy as np
import pytest
import torch

from conftest import assert_close
from testutil import random_model, simulate_obs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def aux():
    from paper_2303_00301_b200 import _lib, auxk, bench_models
    assert _lib.load().auxmc_device_ok() == 1
    return auxk, bench_models


def _run_both(oracle, auxk, otg, gtg, x0, delta, seed, C, steps, backend, adapt=None):
    ch = auxk.init_chains(gtg, x0, delta, seed, C)
    root = oracle.from_seed(seed)
    ochains = [oracle.AuxChain(otg, x0, delta) for _ in range(C)]
    assert_close(ch.log_gamma.cpu(), [o.c.log_gamma for o in ochains], 1e-10, "init log_gamma")
    for it in range(steps):
        ch.kernel_step(backend)
        for c, o in enumerate(ochains):
            o.step(oracle.derive(root, oracle.L_CHAIN, c), backend)
        if adapt is not None:
            ch.adapt_delta(adapt)
            for o in ochains:
                o.adapt(adapt)
        acc = ch.accepted.cpu().numpy()
        oacc = np.array([o.c.stats.accepted for o in ochains])
        assert np.array_equal(acc, oacc), f"step {it}: accepted {acc} vs oracle {oacc}"
        la = ch.last_log_alpha.cpu().numpy()
        ola = np.array([o.c.stats.last_log_alpha for o in ochains])
        fin = np.isfinite(ola)
        assert np.array_equal(np.isfinite(la), fin)
        assert np.all(np.abs(la[fin] - ola[fin]) <= 1e-7 * np.maximum(1.0, np.abs(ola[fin]))), \
            f"step {it}: log alpha {la} vs {ola}"
    x = ch.x.cpu().numpy()
    for c, o in enumerate(ochains):
        assert_close(x[c], o.x, 1e-9, f"chain {c} path")
        assert_close(ch.log_gamma[c].cpu(), o.c.log_gamma, 1e-9, "log_gamma")
        assert_close(ch.delta[c].cpu(), o.c.delta, 1e-12, "delta")
    return ch, ochains


@pytest.mark.parametrize("backend", [0, 1, 2])
def test_exact_lgssm_target_unit_acceptance(aux, oracle, backend):
    auxk, bm = aux
    s = oracle.spec("lgssm-synthetic", T=10, dx=2, dy=1, data_seed=3)
    lat, data = oracle.simulate(s)
    otg = oracle.make_target(s, data)
    gtg = auxk.make_target(bm.ModelSpec(kind="lgssm-synthetic", T=10, dx=2, dy=1, data_seed=3), data)
    x0 = np.tile(otg.arrays()["m0"], (11, 1))
    ch, _ = _run_both(oracle, auxk, otg, gtg, x0, 0.8, 99, 3, 8, backend)
    assert np.all(np.abs(ch.last_log_alpha.cpu().numpy()) < 1e-8)
    assert int(ch.accepted.sum()) == 3 * 8


@pytest.mark.parametrize("backend", [0, 1, 2])
def test_generic_gaussian_potentials(aux, oracle, backend):
    auxk, _ = aux
    s = oracle.derive(oracle.from_seed(12), oracle.L_SIMULATE, 2)
    m = random_model(s, 15, 2, 1, time_varying=True, with_mask=True)
    obs = simulate_obs(m, oracle.from_seed(13))
    otg = oracle.target_from_lgssm(m, obs, generic=True)
    gtg = auxk.GenSSMTarget.linear_generic(m, obs)
    x0 = np.tile(m.m0, (16, 1))
    _run_both(oracle, auxk, otg, gtg, x0, 0.7, 5, 4, 10, backend)


def test_masked_time_varying_exact_target(aux, oracle):
    auxk, _ = aux
    s = oracle.derive(oracle.from_seed(21), oracle.L_SIMULATE, 2)
    m = random_model(s, 12, 3, 2, time_varying=True, with_mask=True)
    obs = simulate_obs(m, oracle.from_seed(22))
    otg = oracle.target_from_lgssm(m, obs, generic=False)
    gtg = auxk.GenSSMTarget.linear_exact(m, obs)
    x0 = np.tile(m.m0, (13, 1))
    ch, _ = _run_both(oracle, auxk, otg, gtg, x0, 0.5, 8, 3, 6, 0)
    assert np.all(np.abs(ch.last_log_alpha.cpu().numpy()) < 1e-8)


@pytest.mark.parametrize("kind,kw,delta,steps,backend", [
    ("stochvol", dict(dx=3, data_seed=11), 1.0, 12, 1),
    ("spatio-temporal", dict(grid=3, data_seed=7), 0.5, 8, 0),
    ("grid-1d-test", dict(), 0.5, 12, 2),
    ("diffusion-smoothing", dict(data_seed=3), 0.05, 8, 0),
    ("lorenz96", dict(dx=8, data_seed=3), 0.05, 6, 0),
])
def test_bench_models_match_oracle(aux, oracle, kind, kw, delta, steps, backend):
    auxk, bm = aux
    T = 20
    so = oracle.spec(kind, T=T, **kw)
    lat, data = oracle.simulate(so)
    otg = oracle.make_target(so, data)
    gtg = auxk.make_target(bm.ModelSpec(kind=kind, T=T, **kw), data)
    x0 = lat.copy()
    _run_both(oracle, auxk, otg, gtg, x0, delta, 1, 3, steps, backend,
              adapt=0.574 if kind == "stochvol" else None)


def test_lorenz96_d40_short(aux, oracle):
    """C3 model class at d = 40 (block-cooperative filter path)."""
    auxk, bm = aux
    T = 12
    so = oracle.spec("lorenz96", T=T, dx=40, data_seed=3)
    lat, data = oracle.simulate(so)
    otg = oracle.make_target(so, data)
    gtg = auxk.make_target(bm.ModelSpec(kind="lorenz96", T=T, dx=40, data_seed=3), data)
    _run_both(oracle, auxk, otg, gtg, lat.copy(), 0.05, 1, 2, 3, 0)


def test_log_gamma_and_grad_match_oracle(aux, oracle):
    auxk, bm = aux
    so = oracle.spec("stochvol", T=30, dx=3, data_seed=11)
    lat, data = oracle.simulate(so)
    otg = oracle.make_target(so, data)
    gtg = auxk.make_target(bm.ModelSpec(kind="stochvol", T=30, dx=3, data_seed=11), data)
    paths = np.stack([lat, lat + 0.1, lat - 0.2])
    got = gtg.log_gamma(paths).cpu().numpy()
    want = [otg.log_gamma(p) for p in paths]
    assert_close(got, want, 1e-10, "log_gamma")


@pytest.mark.parametrize("backend", [0, 1])
def test_parallel_filter_option(aux, oracle, backend):
    """KernelOptions::parallel_filter (auxk.cpp:143-146): scan filter inside the step."""
    auxk, bm = aux
    so = oracle.spec("stochvol", T=30, dx=3, data_seed=11)
    lat, data = oracle.simulate(so)
    otg = oracle.make_target(so, data)
    gtg = auxk.make_target(bm.ModelSpec(kind="stochvol", T=30, dx=3, data_seed=11), data)
    ch = auxk.init_chains(gtg, lat, 1.0, 4, 3)
    oc = [oracle.AuxChain(otg, lat, 1.0) for _ in range(3)]
    root = oracle.from_seed(4)
    for it in range(6):
        ch.kernel_step(backend, parallel_filter=True)
        for c, o in enumerate(oc):
            o.step(oracle.derive(root, oracle.L_CHAIN, c), backend, 1)
        assert np.array_equal(ch.accepted.cpu().numpy(), [o.c.stats.accepted for o in oc])
    for c, o in enumerate(oc):
        assert_close(ch.x[c].cpu().numpy(), o.x, 1e-8, "path")


@pytest.mark.parametrize("backend", [1, 2])
def test_parallel_filter_option_spatio_temporal_d9(aux, oracle, backend):
    """C5 class at small T: spatio-temporal grid 3 (d = 9), scan filter inside the
    aux-K step, prefix / DnC backends (group kernels for d > 8)."""
    auxk, bm = aux
    so = oracle.spec("spatio-temporal", T=24, grid=3, data_seed=7)
    lat, data = oracle.simulate(so)
    otg = oracle.make_target(so, data)
    gtg = auxk.make_target(bm.ModelSpec(kind="spatio-temporal", T=24, grid=3, data_seed=7), data)
    ch = auxk.init_chains(gtg, lat, 0.5, 6, 2)
    oc = [oracle.AuxChain(otg, lat, 0.5) for _ in range(2)]
    root = oracle.from_seed(6)
    for it in range(4):
        ch.kernel_step(backend, parallel_filter=True)
        for c, o in enumerate(oc):
            o.step(oracle.derive(root, oracle.L_CHAIN, c), backend, 1)
        assert np.array_equal(ch.accepted.cpu().numpy(), [o.c.stats.accepted for o in oc])
    for c, o in enumerate(oc):
        assert_close(ch.x[c].cpu().numpy(), o.x, 1e-8, "path")


@pytest.mark.parametrize("backend", [0, 1, 2])
def test_sharded_chains_equal_unsharded(aux, backend):
    """Multi-GPU sharding contract: chain c depends only on its global index, so
    running chains [0,2) and [2,4) separately (two ranks) reproduces one batch
    of 4 bit for bit."""
    auxk, bm = aux
    spec = bm.ModelSpec(kind="stochvol", T=20, dx=3, data_seed=11)
    lat, data = bm.simulate(spec)
    tg = auxk.make_target(spec, data)
    full = auxk.init_chains(tg, lat, 0.5, 3, 4)
    parts = [auxk.init_chains(tg, lat, 0.5, 3, 2, first=f) for f in (0, 2)]
    for _ in range(3):
        full.kernel_step(backend)
        for p in parts:
            p.kernel_step(backend)
    assert torch.equal(torch.cat([p.x for p in parts]), full.x)
    assert torch.equal(torch.cat([p.accepted for p in parts]), full.accepted)


@pytest.mark.parametrize("kind,kw,backend,pf", [
    ("lgssm-synthetic", dict(dx=1, dy=1, data_seed=1), 1, True),   # C1 shape
    ("stochvol", dict(dx=3, data_seed=11), 0, False),
    ("stochvol", dict(dx=3, data_seed=11), 2, False),
])
def test_graph_step_bit_equal_to_eager(aux, kind, kw, backend, pf):
    """AuxChains.graph_step (one CUDA graph per step) reproduces eager kernel_step
    bit for bit, step after step (device-side iteration counters)."""
    auxk, bm = aux
    spec = bm.ModelSpec(kind=kind, T=40, **kw)
    lat, data = bm.simulate(spec)
    tg = auxk.make_target(spec, data)
    x0 = lat if kind != "lgssm-synthetic" else np.tile(tg.m0.cpu().numpy(), (41, 1))
    a = auxk.init_chains(tg, x0, 0.7, 5, 3)
    b = auxk.init_chains(tg, x0, 0.7, 5, 3)
    for _ in range(5):
        a.kernel_step(backend, parallel_filter=pf)
        b.graph_step(backend, parallel_filter=pf)
    torch.cuda.synchronize()
    assert b.graph_launches(backend, parallel_filter=pf) > 5
    assert torch.equal(a.x, b.x)
    assert torch.equal(a.log_gamma, b.log_gamma)
    assert torch.equal(a.accepted, b.accepted)
    assert torch.equal(a.iter, b.iter)
