"""The scan filter's covariance fixed point (pfilter_gen.cu, bc_chain_step and the
recovery's factor reuse).  For a model whose F, Q, H, R are shared by every step
the filtered covariance follows the same map at every step; once a prefix chain
returns its covariance unchanged, later steps only move the means.  The fixed-point
form must give the bits of the full form (auxmc_test_pfg_fixed_point(0)), and the
full form matches the oracle's scan elsewhere (test_gpu_lgssm.py)."""
import numpy as np
import pytest
import torch

from conftest import assert_close
from testutil import predrawn, to_gpu_model

pytestmark = pytest.mark.gpu

FIELDS = ("filt_mean", "filt_cov", "pred_mean", "pred_cov", "log_marginal")


@pytest.fixture(scope="module")
def mods():
    from paper_2303_00301_b200 import _lib, auxk, bench_models as bm, lgssm
    lib = _lib.load()
    assert lib.auxmc_device_ok() == 1
    yield lib, lgssm, auxk, bm
    lib.auxmc_test_pfg_fixed_point(1)


def _strong_model(oracle, T, d, dy, r, seed):
    """Oracle-layout model with F, Q, H, R shared by every step (time-invariant) and
    observation noise r: small r drives the filtered covariance to its fixed point
    within a few steps."""
    rng = np.random.default_rng(seed)
    F = 0.8 * np.eye(d) + 0.05 * rng.standard_normal((d, d))
    F *= 0.9 / np.abs(np.linalg.eigvals(F)).max()  # stable: the data stay O(1)
    A = rng.standard_normal((d, d))
    Q = 0.1 * np.eye(d) + 0.01 * A @ A.T
    H = np.eye(dy, d) + 0.1 * rng.standard_normal((dy, d))
    R = r * np.eye(dy)
    b = 0.1 * rng.standard_normal(d)
    m = oracle.Model.homogeneous(T, rng.standard_normal(d), np.eye(d), F, b, Q, H, np.zeros(dy), R)
    x = np.zeros(d)
    obs = np.zeros((T + 1, dy))
    for t in range(T + 1):
        obs[t] = H @ x + np.sqrt(r) * rng.standard_normal(dy)
        x = F @ x + b + rng.multivariate_normal(np.zeros(d), Q)
    return m, obs


def _both(lib, fn):
    out = []
    try:
        for on in (0, 1):
            lib.auxmc_test_pfg_fixed_point(on)
            lib.auxmc_test_pfg_fixed_point_steps(1)
            r = fn()
            torch.cuda.synchronize()
            out.append((r, lib.auxmc_test_pfg_fixed_point_steps(1)))
    finally:
        lib.auxmc_test_pfg_fixed_point(1)
    return out


@pytest.mark.parametrize("T,d,dy,r", [(5000, 16, 16, 1e-3), (3000, 10, 3, 1e-2), (700, 16, 4, 1.0),
                                      (2500, 20, 20, 1e-3)])
def test_fixed_point_filter_bit_identical(mods, oracle, T, d, dy, r):
    """Warp groups (d <= 16, one and two carry levels) and CTA groups (d = 20)."""
    lib, lgssm, _, _ = mods
    m, obs = _strong_model(oracle, T, d, dy, r, seed=T + d)
    gm = to_gpu_model(m)
    (full, n_full), (fixed, n_fixed) = _both(lib, lambda: lgssm.parallel_filter(gm, obs))
    assert n_full == 0
    assert n_fixed > 0, "no chain reached a covariance fixed point"
    for name in FIELDS:
        assert torch.equal(getattr(full, name), getattr(fixed, name)), name
    # backward elements (k_bwd_lean for d >= 16: steady-state reuse) under two samplers
    term, back, _ = predrawn(np.random.default_rng(T), 3, T, d)
    noise = lgssm.Noise.predrawn(term, back, None)
    for sampler in (0, 1):
        draw = lambda: lgssm.PathSampler(gm, 3, sampler, True)(fixed, noise)  # noqa: E731
        (p_full, _), (p_fixed, _) = _both(lib, draw)
        assert torch.equal(p_full, p_fixed), f"sampler {sampler}"
    want = oracle.kalman_filter(m, obs)
    assert_close(fixed.filt_mean[0].cpu(), want.filt_mean, 1e-8, "filt_mean vs oracle")
    assert_close(fixed.filt_cov[0].cpu(), want.filt_cov, 1e-8, "filt_cov vs oracle")
    assert_close(fixed.log_marginal[0].cpu(), want.log_marginal, 1e-9, "log_marginal vs oracle")


def test_time_varying_model_takes_full_steps(mods, oracle):
    """Per-step matrices (even with equal values) never take the vector-only form."""
    lib, lgssm, _, _ = mods
    m, obs = _strong_model(oracle, 600, 16, 16, 1e-3, seed=3)
    T = m.T
    rep = lambda a, n: np.repeat(a, n, axis=0)  # noqa: E731
    per = lgssm.Model(T, m.m0, m.P0, rep(m.F, T), rep(m.b, T), rep(m.Q, T), rep(m.H, T + 1),
                      rep(m.c, T + 1), rep(m.R, T + 1), None)
    lib.auxmc_test_pfg_fixed_point_steps(1)
    a = lgssm.parallel_filter(per, obs)
    torch.cuda.synchronize()
    assert lib.auxmc_test_pfg_fixed_point_steps(1) == 0
    b = lgssm.parallel_filter(to_gpu_model(m), obs)
    for name in FIELDS:
        assert torch.equal(getattr(a, name), getattr(b, name)), name


def test_c5_shape_aux_step_bit_identical(mods):
    """The C5 aux-Kalman step (spatio-temporal d = 16, scan filter + prefix sampler)
    at T = 2^14: identical decisions, log alpha and paths with the form on and off."""
    lib, _, auxk, bm = mods
    spec = bm.ModelSpec(kind="spatio-temporal", T=1 << 14, grid=4, data_seed=7)
    lat, data = bm.simulate(spec)
    tg = auxk.make_target(spec, data)

    def run():
        ch = auxk.init_chains(tg, lat, 5e-4, 1, 1)
        hist = []
        for _ in range(2):
            ch.kernel_step(auxk.Backend.kPrefix, parallel_filter=True)
            hist.append((ch.accepted.cpu().clone(), ch.last_log_alpha.cpu().clone(),
                         ch.x.cpu().clone()))
        return hist

    (full, _), (fixed, n_fixed) = _both(lib, run)
    assert n_fixed > 0
    for (a0, l0, x0), (a1, l1, x1) in zip(full, fixed):
        assert torch.equal(a0, a1) and torch.equal(l0, l1) and torch.equal(x0, x1)


def test_long_row_sums_keep_their_order(mods, oracle):
    """Few long rows are summed in two kernels (k_sum_parts: chunk sums by warps of many
    CTAs, then cta_sum_fixed's tree): the bits of the one-CTA-per-row form, which runs
    for 17 rows.  Scan-filter log p(y) (d = 7) and the path density, T = 70000."""
    lib, lgssm, _, _ = mods
    T, d, dy = 70000, 7, 2
    m, obs = _strong_model(oracle, T, d, dy, 0.1, seed=5)
    gm = to_gpu_model(m)
    one = lgssm.parallel_filter(gm, obs)
    many = lgssm.parallel_filter(gm, np.stack([obs] * 17))
    assert torch.equal(one.log_marginal[0], many.log_marginal[0])
    assert torch.equal(many.log_marginal, many.log_marginal[:1].expand(17))
    traj = one.filt_mean[0]
    lp1 = lgssm.path_logpdf(gm, obs, traj, one)
    lp17 = lgssm.path_logpdf(gm, obs, traj.expand(17, -1, -1).contiguous(), one)
    assert torch.equal(lp1[0], lp17[0]) and torch.equal(lp17, lp17[:1].expand(17))
