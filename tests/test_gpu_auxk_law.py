"""Law-level GPU tests of the auxiliary Kalman sampler with many chains at once.

The reference checks invariance with 10 000 independent chains of 10 steps run
one after another (test_target_auxk.cpp:256-290) and long-run marginals of the
nonlinear 1-d models against an exact grid recursion (test_target_auxk.cpp:233-254,
acceptance.cpp:168-200).  On the device both are one batch of chains:
  * chains started at exact posterior draws stay at the posterior after 10
    partially accepted steps (every backend, both filters);
  * the grid-1d-test model (quartic potential, no Gaussian closed form): pooled
    chain means match bench::grid_hmm_posterior within 4 standard errors.
"""
import numpy as np
import pytest
import torch

from testutil import random_model, simulate_obs, to_gpu_model

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gpu():
    from paper_2303_00301_b200 import _lib, auxk, bench_models, lgssm, rng
    assert _lib.load().auxmc_device_ok() == 1
    return auxk, bench_models, lgssm, rng


@pytest.mark.parametrize("backend,pf", [(0, False), (1, False), (2, False), (1, True)])
def test_partial_acceptance_leaves_posterior_invariant(gpu, oracle, backend, pf):
    """test_target_auxk.cpp:256-290 as one batch of 10 000 chains."""
    auxk, _, lgssm, rng = gpu
    s = oracle.derive(oracle.from_seed(8), oracle.L_SIMULATE, 3)
    m = random_model(s, 3, 1, 1)
    obs = simulate_obs(m, oracle.from_seed(81))
    gm = to_gpu_model(m)
    fr = lgssm.kalman_filter(gm, obs)
    C, steps = 10000, 10
    roots = rng.chain_keys(800, C)
    # x0_c = backward_sample(m, fr, cr.derive(kSimulate, 0)) on the device
    init = np.array([oracle.derive(oracle.derive(oracle.from_seed(800), oracle.L_CHAIN, c),
                                   oracle.L_SIMULATE, 0).key for c in range(C)], np.uint64)
    x0 = lgssm.PathSampler(gm, C, 0, True)(fr, lgssm.Noise.stream(
        torch.from_numpy(init.view(np.int64)).cuda()))
    tg = auxk.GenSSMTarget.linear_generic(m, obs)
    ch = auxk.AuxChains(tg, x0, 0.8, roots)
    for _ in range(steps):
        ch.kernel_step(backend, parallel_filter=pf)
    acc = int(ch.accepted.sum())
    assert 0 < acc < C * steps, "the gradient linearization is inexact here: some rejections"
    assert int(ch.aborted.sum()) == 0
    mean, cov, _ = oracle.dense_oracle(m, obs)
    fin = ch.x[:, :, 0].cpu().numpy()
    n = float(C)
    for t in range(4):
        mu, var = mean[t], cov[t, t]
        col = fin[:, t]
        mh, vh = col.mean(), col.var(ddof=1)
        assert abs(mh - mu) < 4.0 * np.sqrt(var / n), (t, mh, mu)
        assert abs(vh - var) < 4.0 * np.sqrt(2.0 / (n - 1.0)) * var, (t, vh, var)


def test_grid_model_marginals_match_grid_recursion(gpu, oracle):
    """acceptance.cpp:168-200 (crit_grid_oracle): nonlinear 1-d posterior vs an
    independent grid oracle, here pooled over 2048 chains after adaptation."""
    auxk, bm, _, rng = gpu
    T = 10
    so = oracle.spec("grid-1d-test", T=T)
    _, data = oracle.simulate(so)
    otg = oracle.make_target(so, data)
    _, _, gmean, _, _ = oracle.grid_hmm_posterior(otg, -4.0, 4.0, 2000)
    tg = auxk.make_target(bm.ModelSpec(kind="grid-1d-test", T=T), data)
    C, burn, keep = 2048, 300, 200
    ch = auxk.AuxChains(tg, np.zeros((T + 1, 1)), 1.0, rng.chain_keys(401, C))
    for _ in range(burn):
        ch.kernel_step(auxk.Backend.kSequential)
        ch.adapt_delta(0.574)
    sums = torch.zeros((C, T + 1), dtype=torch.float64, device="cuda")
    for _ in range(keep):
        ch.kernel_step(auxk.Backend.kSequential)
        sums += ch.x[:, :, 0]
    cm = (sums / keep).cpu().numpy()      # per-chain means (independent across chains)
    se = cm.std(axis=0, ddof=1) / np.sqrt(C)
    z = np.abs(cm.mean(axis=0) - gmean) / se
    assert np.all(z < 4.0), z
    rate = int(ch.accepted.sum()) / float(C * (burn + keep))
    assert 0.3 < rate < 0.95, rate
