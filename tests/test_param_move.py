"""Diffusion-coefficient RW-MH within Gibbs (bench/runner.cpp:61-85).

CPU: the oracle's `ao_gamma_move` against a numpy restatement of runner.cpp:61-85
(Lorenz-63 drift from models.cpp:70-85, stream root.derive(kParam, iter)).
GPU: `auxmc_gamma_move` against the oracle for Lorenz-63 and Lorenz-96 batches —
accept flags identical, γ to 1e-12 (libdevice log/exp/cos vs glibc: ≤ 1 ulp) — and a
law-level check: with the path fixed, many independent γ chains reproduce the
posterior mean of log γ computed by quadrature.
"""
import math

import numpy as np
import pytest
import torch

from conftest import assert_close


def _l63_mean(s, x):
    f = np.array([s.lz_sigma * (x[1] - x[0]), x[0] * (s.lz_rho - x[2]) - x[1],
                  x[0] * x[1] - s.lz_beta * x[2]])
    return x + s.lz_h * f


def _numpy_gamma_move(s, x, gamma, step, stream, oracle):
    T = x.shape[0] - 1
    sse = 0.0
    for t in range(T):
        r = x[t + 1] - _l63_mean(s, x[t])
        sse += float(r @ r)
    h = s.lz_h
    ll = lambda g: -1.5 * T * math.log(2.0 * math.pi * h * g * g) - sse / (2.0 * h * g * g)
    lg = math.log(gamma)
    lgp = lg + step * oracle.next_normal(stream)
    gp = math.exp(lgp)
    log_r = ll(gp) - 0.5 * lgp * lgp - (ll(gamma) - 0.5 * lg * lg)
    if math.log(oracle.next_uniform(stream)) < log_r:
        return gp, True
    return gamma, False


def test_oracle_gamma_move_matches_runner(oracle):
    so = oracle.spec("diffusion-smoothing", T=60, data_seed=3)
    lat, data = oracle.simulate(so)
    otg = oracle.make_target(so, data)
    root = oracle.derive(oracle.from_seed(1), oracle.L_CHAIN, 0)
    moves = 0
    for it, (g, step) in enumerate([(2.0, 0.1), (2.0, 0.5), (1.0, 0.3), (3.5, 0.2), (0.7, 1.0),
                                    (2.2, 0.05), (1.9, 0.8), (5.0, 0.4)]):
        got = oracle.gamma_move(otg, lat, g, step, oracle.derive(root, oracle.L_PARAM, it))
        want = _numpy_gamma_move(so, lat, g, step, oracle.derive(root, oracle.L_PARAM, it), oracle)
        assert got[1] == want[1], it
        assert_close([got[0]], [want[0]], 1e-14, "gamma")
        moves += got[1]
    assert 0 < moves < 8


def _setup(oracle, kind, T, kw):
    from paper_2303_00301_b200 import auxk, bench_models as bm
    so = oracle.spec(kind, T=T, **kw)
    lat, data = oracle.simulate(so)
    otg = oracle.make_target(so, data)
    gtg = auxk.make_target(bm.ModelSpec(kind=kind, T=T, **kw), data)
    return so, lat, otg, gtg


@pytest.mark.gpu
@pytest.mark.parametrize("kind,T,kw", [("diffusion-smoothing", 100, dict(data_seed=3)),
                                       ("diffusion-smoothing", 7, dict(data_seed=5)),
                                       ("lorenz96", 50, dict(dx=8, data_seed=3)),
                                       ("lorenz96", 33, dict(dx=40, data_seed=3))])
def test_gpu_gamma_move_matches_oracle(oracle, kind, T, kw):
    from paper_2303_00301_b200 import auxk
    from paper_2303_00301_b200.rng import chain_keys
    so, lat, otg, gtg = _setup(oracle, kind, T, kw)
    C = 96
    rs = np.random.default_rng(4)
    paths = lat[None] + 0.02 * rs.standard_normal((C,) + lat.shape)
    gam = np.exp(rs.uniform(-1.5, 2.0, C))
    keys = chain_keys(7, C)
    g_dev, moved_dev = torch.as_tensor(gam, device="cuda"), None
    g_or = gam.copy()
    for it in range(5):
        step = [0.05, 0.3, 1.0, 0.1, 0.6][it]
        g_dev, moved_dev = auxk.gamma_move(gtg, paths, keys, it, step, g_dev)
        mv = moved_dev.cpu().numpy()
        for c in range(C):
            st = oracle.derive(oracle.derive(oracle.from_seed(7), oracle.L_CHAIN, c), oracle.L_PARAM, it)
            g_or[c], m = oracle.gamma_move(otg, paths[c], g_or[c], step, st)
            assert bool(mv[c]) == m, (it, c)
        assert_close(g_dev.cpu().numpy(), g_or, 1e-12, "gamma")


@pytest.mark.gpu
def test_gpu_gamma_move_posterior_law(oracle):
    """Fixed path: C independent γ chains; E[log γ | x] by quadrature over log γ."""
    from paper_2303_00301_b200 import auxk
    from paper_2303_00301_b200.rng import chain_keys
    T = 40
    so, lat, otg, gtg = _setup(oracle, "diffusion-smoothing", T, dict(data_seed=3))
    sse = sum(float(np.sum((lat[t + 1] - _l63_mean(so, lat[t])) ** 2)) for t in range(T))
    h = so.lz_h
    lg = np.linspace(-6, 6, 200001)
    g = np.exp(lg)
    lp = -1.5 * T * np.log(2 * np.pi * h * g * g) - sse / (2 * h * g * g) - 0.5 * lg * lg
    w = np.exp(lp - lp.max())
    mean = float(np.sum(w * lg) / np.sum(w))
    sd = math.sqrt(float(np.sum(w * (lg - mean) ** 2) / np.sum(w)))
    C = 20000
    keys = chain_keys(11, C)
    x = torch.as_tensor(np.broadcast_to(lat, (C,) + lat.shape).copy(), device="cuda")
    gam = torch.full((C,), 2.0, dtype=torch.float64, device="cuda")
    acc = 0
    for it in range(300):
        gam, m = auxk.gamma_move(gtg, x, keys, it, 2.4 * sd, gam)
        acc += int(m.sum())
    est = gam.log().cpu().numpy()
    se = sd / math.sqrt(C)
    assert abs(est.mean() - mean) < 6 * se, (est.mean(), mean, se)
    assert abs(est.std() - sd) < 0.05 * sd, (est.std(), sd)
    assert 0.1 < acc / (300 * C) < 0.9


@pytest.mark.gpu
def test_gpu_gamma_move_rejects_linear_target(oracle):
    from paper_2303_00301_b200 import auxk, _lib
    from paper_2303_00301_b200.rng import chain_keys
    so, lat, otg, gtg = _setup(oracle, "stochvol", 10, dict(dx=3, data_seed=11))
    with pytest.raises(Exception):
        auxk.gamma_move(gtg, lat, chain_keys(1, 1), 0, 0.1, 1.0)
