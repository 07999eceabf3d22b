"""Pseudo-marginal potentials (fkpg.cpp:233-250 pm_potential) in the device particle Gibbs,
with the estimators of the reference's own tests (auxmc_gpu.h AUXMC_PM_*), against the
reference itself (oracle/_ref: aux_pgibbs_step with PgOptions::fk_transform).

  zero variance      test_fkpg.cpp:365-381: an exact estimator changes no draw
  unbiased noise     acceptance.cpp:249-290 / test_fkpg.cpp:402-434: the two-point
                     multiplicative noise keeps the posterior; same draws as _ref
  contract           test_fkpg.cpp:436-445: a negative estimate is a ContractError
"""
import numpy as np
import pytest
import torch

from conftest import assert_close
from testutil import random_model, simulate_obs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    from paper_2303_00301_b200 import _lib, auxk, fkpg, rng
    assert _lib.load().auxmc_device_ok() == 1
    return _lib, auxk, fkpg, rng


@pytest.fixture(scope="module")
def ref():
    from oracle import refbridge as R
    if not R.available():
        pytest.skip("oracle/_ref not built")
    return R


def _case(oracle, seed, T):
    s = oracle.derive(oracle.from_seed(seed), oracle.L_SIMULATE, 8)
    m = random_model(s, T, 1, 1)
    obs = simulate_obs(m, oracle.from_seed(seed * 10 + 1))
    return m, obs


def _root(oracle, seed, c=0):
    k = oracle.derive(oracle.from_seed(seed), oracle.L_CHAIN, c).key
    return torch.tensor([k], dtype=torch.uint64).view(torch.int64).cuda()


def test_two_point_estimator_matches_reference(mods, oracle, ref):
    """Prior-mode pgibbs on the generic LGSSM target (the reference test's setting), two-
    point noisy potentials: every iteration's path and aux keys equal the reference's."""
    _lib, auxk, fkpg, _ = mods
    m, obs = _case(oracle, 16, 3)
    gtg = auxk.GenSSMTarget.linear_generic(m, obs)
    rtg = ref.target_from_lgssm(m, obs, generic=True)
    x0 = np.zeros((4, 1))
    ch = fkpg.PGChains(gtg, x0, 1.0, _root(oracle, 162), 8, pm=fkpg.PseudoMarginal.kTwoPoint)
    rp = ref.PGChain(rtg, x0, 1.0)
    root = oracle.derive(oracle.from_seed(162), oracle.L_CHAIN, 0)
    for it in range(40):
        ch.aux_pgibbs_step(fkpg.Variant.kReference, fkpg.ProposalMode.kPrior)
        st, bad = rp.step(8, root, mode=0, pm=fkpg.PseudoMarginal.kTwoPoint)
        assert st == 0 and int(ch.status[0]) == 0
        s = rp.state()
        assert np.array_equal(ch.keys[0].cpu().numpy().view(np.uint64), s["keys"]), f"keys {it}"
        assert_close(ch.x[0].cpu().numpy(), s["x"], 1e-12, f"path {it}")
        assert int(ch.updates[0]) == s["updates"]


def test_exact_estimator_changes_no_draw(mods, oracle):
    _lib, auxk, fkpg, _ = mods
    m, obs = _case(oracle, 13, 4)
    gtg = auxk.GenSSMTarget.linear_generic(m, obs)
    x0 = np.zeros((5, 1))
    a = fkpg.PGChains(gtg, x0, 1.0, _root(oracle, 14), 8)
    b = fkpg.PGChains(gtg, x0, 1.0, _root(oracle, 14), 8, pm=fkpg.PseudoMarginal.kExact)
    for _ in range(10):
        a.aux_pgibbs_step(fkpg.Variant.kReference, fkpg.ProposalMode.kPrior)
        b.aux_pgibbs_step(fkpg.Variant.kReference, fkpg.ProposalMode.kPrior)
        assert torch.equal(a.x, b.x)
        assert torch.equal(a.keys, b.keys)


def test_negative_estimate_is_a_contract_error(mods, oracle, ref):
    _lib, auxk, fkpg, _ = mods
    m, obs = _case(oracle, 17, 2)
    gtg = auxk.GenSSMTarget.linear_generic(m, obs)
    ch = fkpg.PGChains(gtg, np.zeros((3, 1)), 1.0, _root(oracle, 18), 4,
                       pm=fkpg.PseudoMarginal.kNegative)
    ch.aux_pgibbs_step(fkpg.Variant.kReference, fkpg.ProposalMode.kPrior)
    assert int(ch.status[0]) == _lib.E_CONTRACT and int(ch.bad_t[0]) == 0
    rp = ref.PGChain(ref.target_from_lgssm(m, obs, generic=True), np.zeros((3, 1)), 1.0)
    st, _ = rp.step(4, oracle.from_seed(18), mode=0, pm=fkpg.PseudoMarginal.kNegative)
    assert st == ref.RB_E_CONTRACT
    # the PIT variant has no pseudo-marginal form: refused
    ch2 = fkpg.PGChains(gtg, np.zeros((3, 1)), 1.0, _root(oracle, 18), 4,
                        pm=fkpg.PseudoMarginal.kTwoPoint)
    with pytest.raises(_lib.AuxmcError):
        ch2.aux_pgibbs_step(fkpg.Variant.kPit, fkpg.ProposalMode.kGradient)


def test_noisy_potentials_keep_the_posterior(mods, oracle):
    """acceptance.cpp:249-290 on 4096 independent chains: after burn-in with delta
    adaptation, the chains' states match the smoothed marginals (4 standard errors)."""
    _lib, auxk, fkpg, rng = mods
    m, obs = _case(oracle, 601, 4)
    gtg = auxk.GenSSMTarget.linear_generic(m, obs)
    fr = oracle.kalman_filter(m, obs)
    smean, scov = oracle.rts_smoother(m, fr)
    C = 4096
    ch = fkpg.init_pg(gtg, np.zeros((5, 1)), 1.0, 603, C, 8)
    ch.pm = fkpg.PseudoMarginal.kTwoPoint
    for i in range(400):
        ch.aux_pgibbs_step(fkpg.Variant.kReference, fkpg.ProposalMode.kPrior)
        if i < 200:
            ch.adapt_delta(0.9)
    assert int(ch.status.max()) == 0
    x = ch.x[:, :, 0].cpu().numpy()
    mu, var = smean[:, 0], scov[:, 0, 0]
    z_mean = np.abs(x.mean(0) - mu) / np.sqrt(var / C)
    z_var = np.abs(x.var(0, ddof=1) - var) / (var * np.sqrt(2.0 / (C - 1)))
    assert z_mean.max() < 4.5, z_mean
    assert z_var.max() < 4.5, z_var
