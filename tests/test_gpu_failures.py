"""The reference's failure semantics on the device, mirroring its own tests:

  jitter ladder      test_gauss.cpp:161-173 (gauss.cpp:26-35): rank-1 + 1e-13 takes the
                     1e-10 rung; -I fails with FactorizationError (AUXMC_E_FACTOR)
  abort              test_target_auxk.cpp:374-392 (auxk.cpp:157-162): a non-finite
                     proposal gradient aborts the step
  nonfinite_gamma    test_target_auxk.cpp:394-414 (auxk.cpp:151-155): a proposal outside
                     the support is rejected and counted
  degenerate weights test_fkpg.cpp:447-465 (fkpg.cpp:19-23): all weights -inf at t = 2
                     -> AUXMC_E_DEGENERATE naming t = 2

Each device result is also compared with the reference itself (oracle/_ref) on the same
streams: identical counters and paths.
"""
import numpy as np
import pytest
import torch

from conftest import assert_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    from paper_2303_00301_b200 import _lib, auxk, fkpg, lgssm, pit, rng
    assert _lib.load().auxmc_device_ok() == 1
    return dict(_lib=_lib, auxk=auxk, fkpg=fkpg, lgssm=lgssm, pit=pit, rng=rng)


@pytest.fixture(scope="module")
def ref():
    from oracle import refbridge as R
    if not R.available():
        pytest.skip("oracle/_ref not built")
    return R


def _t0_model(oracle, P0):
    """T = 0, one unobserved step: filt_cov[0] = P0 (lgssm.cpp:86-111)."""
    d = P0.shape[0]
    return oracle.Model(0, np.zeros(d), P0, np.eye(d)[None], np.zeros((1, d)), np.eye(d)[None],
                        np.zeros((1, 1, d)), np.zeros((1, 1)), np.eye(1)[None], mask=[0])


def test_jitter_ladder_first_rung(mods, oracle, ref):
    lgssm, pit = mods["lgssm"], mods["pit"]
    a = np.ones((3, 3))
    a[2, 2] += 1e-13
    om = _t0_model(oracle, a)
    from testutil import to_gpu_model
    gm = to_gpu_model(om)
    fr = lgssm.kalman_filter(gm, np.zeros((1, 1)))
    mean, cov = pit.extract_affine_law(pit.Sampler.kSequential, gm, fr)
    cov = cov.cpu().numpy().reshape(3, 3)
    diff = cov - a
    # L L^T = a + eps s I with s = trace/3: the 1e-10 rung, not the 1e-8 one
    s = np.trace(a) / 3
    assert np.abs(diff).max() < 1e-8
    assert np.allclose(np.diag(diff), 1e-10 * s, rtol=1e-3, atol=0), np.diag(diff)
    # the same draw as the reference (which factors with the same ladder)
    rm = ref.RModel(om)
    rfr = ref.kalman_filter(rm, np.zeros((1, 1)))
    root = oracle.derive(oracle.from_seed(3), oracle.L_CHAIN, 0)
    want = ref.backward_sample(rm, rfr, root)
    keys = torch.tensor([root.key], dtype=torch.uint64).view(torch.int64).cuda()
    got = lgssm.backward_sample(gm, fr, lgssm.Noise.stream(keys))[0].cpu().numpy()
    assert_close(got, want, 1e-9, "terminal draw through the jittered factor")


def test_negative_definite_raises_factorization_error(mods, oracle):
    lgssm, _lib = mods["lgssm"], mods["_lib"]
    from testutil import to_gpu_model
    gm = to_gpu_model(_t0_model(oracle, -np.eye(2)))
    fr = lgssm.kalman_filter(gm, np.zeros((1, 1)))
    keys = torch.zeros(1, dtype=torch.int64, device="cuda")
    with pytest.raises(_lib.AuxmcError) as e:
        lgssm.backward_sample(gm, fr, lgssm.Noise.stream(keys))
    assert e.value.code == _lib.E_FACTOR
    # a zero covariance factors to zero: the draw is the mean (gauss.cpp:47)
    gz = to_gpu_model(_t0_model(oracle, np.zeros((2, 2))))
    frz = lgssm.kalman_filter(gz, np.zeros((1, 1)))
    x = lgssm.backward_sample(gz, frz, lgssm.Noise.stream(keys))
    assert torch.count_nonzero(x) == 0
    # an indefinite observation covariance fails inside the filter's solves
    m = oracle.Model(3, np.zeros(2), np.eye(2), np.eye(2)[None], np.zeros((1, 2)),
                     np.eye(2)[None], np.ones((1, 1, 2)), np.zeros((1, 1)), -np.eye(1)[None] * 5)
    with pytest.raises(_lib.AuxmcError) as e:
        lgssm.kalman_filter(to_gpu_model(m), np.zeros((4, 1)))
    assert e.value.code == _lib.E_FACTOR


def _root_keys(oracle, seed):
    return torch.tensor([oracle.from_seed(seed).key], dtype=torch.uint64).view(torch.int64).cuda()


@pytest.mark.parametrize("backend", [0, 1, 2])
def test_nonfinite_gradient_aborts(mods, oracle, ref, backend):
    auxk = mods["auxk"]
    T = 2
    tg = auxk.GenSSMTarget.test_kind("test-abort", T)
    ch = auxk.AuxChains(tg, np.zeros((T + 1, 1)), 8.0, _root_keys(oracle, 12))
    rt = ref.test_target("test-abort", T)
    rc = ref.AuxChain(rt, np.zeros((T + 1, 1)), 8.0)
    for i in range(100):
        ch.kernel_step(backend)
        rc.step(oracle.from_seed(12), backend)
    st = rc.state()
    assert int(ch.aborted[0]) > 0
    assert float(ch.x.abs().max()) <= 0.5
    assert int(ch.aborted[0]) == st["aborted"]
    assert int(ch.accepted[0]) == st["accepted"]
    assert_close(ch.x[0].cpu().numpy(), st["x"], 1e-9, "path")


@pytest.mark.parametrize("backend", [0, 1, 2])
def test_out_of_support_counts_nonfinite_gamma(mods, oracle, ref, backend):
    auxk = mods["auxk"]
    T = 2
    tg = auxk.GenSSMTarget.test_kind("test-support", T)
    ch = auxk.AuxChains(tg, np.zeros((T + 1, 1)), 6.0, _root_keys(oracle, 13))
    rt = ref.test_target("test-support", T)
    rc = ref.AuxChain(rt, np.zeros((T + 1, 1)), 6.0)
    for i in range(200):
        ch.kernel_step(backend)
        rc.step(oracle.from_seed(13), backend)
    st = rc.state()
    assert int(ch.nonfinite_gamma[0]) > 0
    assert float(ch.x.max()) <= 0.4
    assert int(ch.nonfinite_gamma[0]) == st["nonfinite_gamma"]
    assert int(ch.accepted[0]) == st["accepted"]
    assert_close(ch.x[0].cpu().numpy(), st["x"], 1e-9, "path")


@pytest.mark.parametrize("variant", [0, 1])
def test_collapsed_weights_name_the_step(mods, oracle, ref, variant):
    auxk, fkpg, _lib = mods["auxk"], mods["fkpg"], mods["_lib"]
    T, N = 3, 8
    tg = auxk.GenSSMTarget.test_kind("test-collapse", T)
    ch = fkpg.PGChains(tg, np.zeros((T + 1, 1)), 1.0, _root_keys(oracle, 19), N)
    ch.aux_pgibbs_step(variant)
    assert int(ch.status[0]) == _lib.E_DEGENERATE
    assert int(ch.bad_t[0]) == 2
    rp = ref.PGChain(ref.test_target("test-collapse", T), np.zeros((T + 1, 1)), 1.0)
    st, bad = rp.step(N, oracle.from_seed(19))
    assert st == ref.RB_E_DEGENERATE and bad == 2
