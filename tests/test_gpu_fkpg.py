"""GPU parity of auxiliary particle Gibbs against the oracle.

Reference variant: ancestor indices and backward (selected) indices must agree
with the oracle's restatement of fkpg.cpp:44-152 exactly, paths bit-for-bit
(they are copies of particles), update counters exactly.  PIT variant: the
oracle's lattice forward-backward sweep with the same streams.
"""
import numpy as np
import pytest
import torch

from conftest import assert_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pg():
    from paper_2303_00301_b200 import _lib, auxk, bench_models, fkpg
    assert _lib.load().auxmc_device_ok() == 1
    return auxk, bench_models, fkpg


def _targets(oracle, auxk, bm, kind, T, kw):
    so = oracle.spec(kind, T=T, **kw)
    lat, data = oracle.simulate(so)
    return lat, oracle.make_target(so, data), auxk.make_target(bm.ModelSpec(kind=kind, T=T, **kw),
                                                              data)


@pytest.mark.parametrize("kind,kw,N", [("stochvol", dict(dx=3, data_seed=11), 16),
                                       ("stochvol", dict(dx=3, data_seed=11), 100),
                                       ("lgssm-synthetic", dict(dx=2, dy=1, data_seed=3), 8),
                                       ("spatio-temporal", dict(grid=2, data_seed=7), 32)])
def test_reference_csmc_indices_bit_exact(pg, oracle, kind, kw, N):
    auxk, bm, fkpg = pg
    T = 25
    lat, otg, gtg = _targets(oracle, auxk, bm, kind, T, kw)
    C = 3
    ch = fkpg.init_pg(gtg, lat, 1.0, 5, C, N, trace=True)
    oc = [oracle.PGChain(otg, lat, 1.0) for _ in range(C)]
    root = oracle.from_seed(5)
    for it in range(4):
        ch.aux_pgibbs_step(fkpg.Variant.kReference)
        anc = ch.ancestors.cpu().numpy()
        sel = ch.selected.cpu().numpy()
        assert int(ch.status.max()) == 0
        for c in range(C):
            st, bad, oanc, osel = oc[c].step(N, oracle.derive(root, oracle.L_CHAIN, c), 1, trace=True)
            assert st == 0
            assert np.array_equal(anc[c], oanc), f"iter {it} chain {c}: ancestors differ"
            assert np.array_equal(sel[c], osel), f"iter {it} chain {c}: backward indices differ"
            assert np.array_equal(ch.x[c].cpu().numpy(), oc[c].x) or \
                np.max(np.abs(ch.x[c].cpu().numpy() - oc[c].x)) < 1e-12
            assert np.array_equal(ch.keys[c].cpu().numpy().view(np.uint64), oc[c].keys)
    assert np.array_equal(ch.updates.cpu().numpy(), [o.p.updates for o in oc])


@pytest.mark.parametrize("mode", [0, 2])  # ProposalMode kPrior, kFullyAdapted
@pytest.mark.parametrize("kind,kw,N", [("stochvol", dict(dx=3, data_seed=11), 16),
                                       ("lgssm-synthetic", dict(dx=2, dy=1, data_seed=3), 8),
                                       ("diffusion-smoothing", dict(data_seed=2), 12)])
def test_reference_csmc_prior_and_adapted_modes(pg, oracle, kind, kw, N, mode):
    """Parent-dependent proposals (fkpg.cpp:154-185): the prior N(dyn_mean, Q) and
    the conjugate fully adapted proposal; ancestors / backward indices exact,
    paths to 1e-9, adapted deltas equal."""
    auxk, bm, fkpg = pg
    T = 20
    lat, otg, gtg = _targets(oracle, auxk, bm, kind, T, kw)
    C = 3
    ch = fkpg.init_pg(gtg, lat, 1.0, 7, C, N, trace=True)
    oc = [oracle.PGChain(otg, lat, 1.0) for _ in range(C)]
    root = oracle.from_seed(7)
    for it in range(3):
        ch.aux_pgibbs_step(fkpg.Variant.kReference, mode=mode)
        ch.adapt_delta(0.9)
        anc = ch.ancestors.cpu().numpy()
        sel = ch.selected.cpu().numpy()
        assert int(ch.status.max()) == 0
        for c in range(C):
            st, bad, oanc, osel = oc[c].step(N, oracle.derive(root, oracle.L_CHAIN, c), mode,
                                             trace=True)
            oc[c].adapt(0.9)
            assert st == 0
            assert np.array_equal(anc[c], oanc), f"iter {it} chain {c}: ancestors differ"
            assert np.array_equal(sel[c], osel), f"iter {it} chain {c}: backward indices differ"
            assert_close(ch.x[c].cpu().numpy(), oc[c].x, 1e-9, f"iter {it} chain {c} path")
    assert np.array_equal(ch.updates.cpu().numpy(), [o.p.updates for o in oc])
    assert_close(ch.delta.cpu().numpy(), [o.p.delta for o in oc], 1e-12, "delta")


def test_pit_variant_rejects_parent_dependent_proposals(pg, oracle):
    auxk, bm, fkpg = pg
    lat, otg, gtg = _targets(oracle, auxk, bm, "stochvol", 8, dict(dx=3, data_seed=11))
    ch = fkpg.init_pg(gtg, lat, 1.0, 1, 1, 8)
    from paper_2303_00301_b200 import _lib
    with pytest.raises(_lib.AuxmcError):
        ch.aux_pgibbs_step(fkpg.Variant.kPit, mode=0)


def test_reference_csmc_single_particle_identity(pg, oracle):
    """test_fkpg.cpp:113-123: N = 1 returns the reference unchanged."""
    auxk, bm, fkpg = pg
    lat, otg, gtg = _targets(oracle, auxk, bm, "stochvol", 12, dict(dx=3, data_seed=11))
    ch = fkpg.init_pg(gtg, lat, 1.0, 1, 2, 1)
    ch.aux_pgibbs_step(fkpg.Variant.kReference)
    assert torch.equal(ch.x[0].cpu(), torch.as_tensor(lat))
    assert int(ch.updates.sum()) == 0


@pytest.mark.parametrize("N", [8, 64])
def test_pit_csmc_matches_oracle(pg, oracle, N):
    auxk, bm, fkpg = pg
    T = 20
    lat, otg, gtg = _targets(oracle, auxk, bm, "stochvol", T, dict(dx=3, data_seed=11))
    C = 3
    ch = fkpg.init_pg(gtg, lat, 1.0, 9, C, N, trace=True)
    oc = [oracle.PGChain(otg, lat, 1.0) for _ in range(C)]
    root = oracle.from_seed(9)
    for it in range(4):
        ch.aux_pgibbs_step(fkpg.Variant.kPit)
        sel = ch.selected.cpu().numpy()
        assert int(ch.status.max()) == 0
        for c in range(C):
            st, bad, osel = oc[c].step_pit(N, oracle.derive(root, oracle.L_CHAIN, c))
            assert st == 0
            assert np.array_equal(sel[c], osel), f"iter {it} chain {c}: indices differ"
            assert_close(ch.x[c].cpu().numpy(), oc[c].x, 1e-12, "path")
    assert np.array_equal(ch.updates.cpu().numpy(), [o.p.updates for o in oc])


def test_pit_csmc_invariance_small_lgssm(pg, oracle):
    """acceptance.cpp:204-244 at law level: PIT particle Gibbs moments match
    the dense posterior (batch-means z < 4.5) on a tiny LGSSM."""
    auxk, bm, fkpg = pg
    s = oracle.spec("lgssm-synthetic", T=3, dx=1, dy=1, data_seed=11)
    lat, data = oracle.simulate(s)
    mean, cov, _ = oracle.dense_oracle(oracle.synthetic_lgssm(s), data)
    gtg = auxk.make_target(bm.ModelSpec(kind="lgssm-synthetic", T=3, dx=1, dy=1, data_seed=11),
                           data)
    C = 512
    ch = fkpg.init_pg(gtg, np.tile(gtg.m0.cpu().numpy(), (4, 1)), 1.0, 3, C, 8)
    for _ in range(20):  # burn-in
        ch.aux_pgibbs_step(fkpg.Variant.kPit)
    draws = []
    for _ in range(60):
        ch.aux_pgibbs_step(fkpg.Variant.kPit)
        draws.append(ch.x[:, :, 0].cpu().numpy().copy())
    draws = np.array(draws)  # [iters, C, 4]
    chain_means = draws.mean(axis=0)  # independent chains -> iid means
    z = np.abs(chain_means.mean(axis=0) - mean) / (chain_means.std(axis=0, ddof=1) / np.sqrt(C))
    assert np.all(z < 4.5), z
