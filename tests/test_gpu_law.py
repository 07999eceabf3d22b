"""GPU law exactness: the device's exact affine law of every pathwise sampler
and its RTS smoother against dense Gaussian conditioning and the oracle.

Mirrors test_pit.cpp:283-337 / runner.cpp:279-312 (`validate`): the law a
sampler induces (pit::extract_affine_law, pit.cpp:303-332 — here one batched
device call pushing every basis noise vector through the kernels) equals the
dense-conditioning posterior to 1e-8, the RTS marginals (lgssm.cpp:114-127)
equal the oracle's and the posterior's diagonal blocks, and a deliberate
backward-gain sign flip (testhooks.hpp:11) makes the law check fail.
"""
import numpy as np
import pytest

from conftest import assert_close
from testutil import random_model, simulate_obs, to_gpu_model

pytestmark = pytest.mark.gpu

CASES = [  # (T, dx, dy, time_varying, with_mask, seed)
    (6, 2, 1, False, False, 1),
    (12, 2, 1, True, True, 2),
    (9, 3, 2, True, False, 3),
    (1, 2, 1, False, False, 4),
    (20, 1, 1, False, True, 5),
    (7, 4, 2, False, False, 6),
]


@pytest.fixture(scope="module")
def gpu():
    from paper_2303_00301_b200 import _lib, lgssm, pit
    assert _lib.load().auxmc_device_ok() == 1
    return _lib, lgssm, pit


def _case(oracle, T, dx, dy, tv, mask, seed):
    s = oracle.derive(oracle.from_seed(seed), oracle.L_SIMULATE, 7)
    m = random_model(s, T, dx, dy, tv, mask)
    obs = simulate_obs(m, oracle.from_seed(300 + seed))
    return m, obs


@pytest.mark.parametrize("which", [0, 1, 2])
@pytest.mark.parametrize("case", CASES)
def test_affine_law_equals_dense_posterior(gpu, oracle, case, which):
    _, lgssm, pit = gpu
    m, obs = _case(oracle, *case)
    gm = to_gpu_model(m)
    fr = lgssm.kalman_filter(gm, obs)
    mean, cov = pit.extract_affine_law(which, gm, fr)
    pm, pc, _ = oracle.dense_oracle(m, obs)
    scale = max(1.0, float(np.abs(pc).max()))
    assert np.abs(mean.cpu().numpy() - pm).max() < 1e-8 * max(1.0, float(np.abs(pm).max()))
    assert np.abs(cov.cpu().numpy() - pc).max() < 1e-8 * scale
    om, oc = oracle.extract_affine_law(which, m, oracle.kalman_filter(m, obs))
    assert_close(mean.cpu().numpy(), om, 1e-9, "law mean vs oracle")
    assert np.abs(cov.cpu().numpy() - oc).max() < 1e-9 * scale


@pytest.mark.parametrize("case", CASES)
def test_rts_smoother_matches_oracle_and_posterior(gpu, oracle, case):
    _, lgssm, _ = gpu
    m, obs = _case(oracle, *case)
    gm = to_gpu_model(m)
    fr = lgssm.kalman_filter(gm, obs)
    mean, cov = lgssm.rts_smoother(gm, fr)
    om, oc = oracle.rts_smoother(m, oracle.kalman_filter(m, obs))
    assert_close(mean[0].cpu().numpy(), om, 1e-9, "rts mean")
    assert_close(cov[0].cpu().numpy(), oc, 1e-9, "rts cov")
    pm, pc, _ = oracle.dense_oracle(m, obs)
    d = m.dx
    for t in range(m.T + 1):
        blk = pc[t * d:(t + 1) * d, t * d:(t + 1) * d]
        assert np.abs(cov[0, t].cpu().numpy() - blk).max() < 1e-8 * max(1.0, np.abs(blk).max())
        assert np.abs(mean[0, t].cpu().numpy() - pm[t * d:(t + 1) * d]).max() < 1e-8 * max(
            1.0, np.abs(pm).max())


def test_rts_smoother_batched_filters(gpu, oracle):
    """Many filter results in one call (the batched form), each equal to its own."""
    _, lgssm, _ = gpu
    m, _ = _case(oracle, 15, 3, 2, False, False, 11)
    obs = np.stack([simulate_obs(m, oracle.from_seed(500 + b)) for b in range(4)])
    gm = to_gpu_model(m)
    fr = lgssm.kalman_filter(gm, obs)
    mean, cov = lgssm.rts_smoother(gm, fr)
    for b in range(4):
        om, oc = oracle.rts_smoother(m, oracle.kalman_filter(m, obs[b]))
        assert_close(mean[b].cpu().numpy(), om, 1e-9, f"rts mean {b}")
        assert_close(cov[b].cpu().numpy(), oc, 1e-9, f"rts cov {b}")


def test_flipped_backward_gain_fails_the_law_check(gpu, oracle):
    """runner.cpp:301-312: the validation suite must catch a wrong backward gain."""
    lib, lgssm, pit = gpu
    m, obs = _case(oracle, *CASES[2])
    gm = to_gpu_model(m)
    fr = lgssm.kalman_filter(gm, obs)
    pm, pc, _ = oracle.dense_oracle(m, obs)
    lib.check(lib.load().auxmc_test_flip_backward_gain(1), "flip")
    try:
        mean, cov = pit.extract_affine_law(1, gm, fr)
    finally:
        lib.check(lib.load().auxmc_test_flip_backward_gain(0), "unflip")
    dev = max(np.abs(mean.cpu().numpy() - pm).max(), np.abs(cov.cpu().numpy() - pc).max())
    assert dev > 1e-3, f"sign-flipped gains still pass the law check (deviation {dev})"
    mean, cov = pit.extract_affine_law(1, gm, fr)  # and the hook is off again
    assert np.abs(cov.cpu().numpy() - pc).max() < 1e-8 * max(1.0, float(np.abs(pc).max()))
