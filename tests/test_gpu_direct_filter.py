"""The structure-aware aux step (filter_direct.cu: fused direct-observation filter; for
Lorenz-96 the dynamics Jacobian as a stencil in the filter, the backward elements and
the path terms) against the generic (d+q)-dimensional path on the same chains
(auxmc_test_force_generic_filter).  Same accept/reject decisions, paths within the
FP64 tolerance, and the reference's failure routing for a target that breaks the
structure contract.  The full-shape C3 test (test_gpu_shapes.py) checks the
structure-aware path against the oracle."""
import numpy as np
import pytest
import torch

from conftest import assert_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    from paper_2303_00301_b200 import _lib, auxk, bench_models as bm
    assert _lib.load().auxmc_device_ok() == 1
    yield _lib, auxk, bm
    _lib.load().auxmc_test_force_generic_filter(0)


def _pair(mods, tg, x0, delta, C, iters, backend=0):
    _lib, auxk, _ = mods
    lib = _lib.load()
    out = []
    lm = torch.zeros(C, dtype=torch.float64, device="cuda")
    lib.auxmc_test_capture_log_marginal(lm.data_ptr())
    try:
        for force in (1, 0):
            lib.auxmc_test_force_generic_filter(force)
            ch = auxk.init_chains(tg, x0, delta, 5, C)
            hist = []
            for _ in range(iters):
                ch.kernel_step(backend)
                hist.append((ch.accepted.cpu().numpy().copy(),
                             ch.last_log_alpha.cpu().numpy().copy(), ch.x.cpu().numpy().copy(),
                             int(ch.aborted.sum()), lm.cpu().numpy().copy()))
            out.append(hist)
    finally:
        lib.auxmc_test_force_generic_filter(0)
        lib.auxmc_test_capture_log_marginal(None)
    return out


def _compare(gen, fused, what):
    for it, ((a0, l0, x0, ab0, m0), (a1, l1, x1, ab1, m1)) in enumerate(zip(gen, fused)):
        assert ab0 == ab1 == 0, f"{what} aborted at {it}"
        # the filters' own output: log p(z) of the forward auxiliary model
        assert_close(m1, m0, 1e-10, f"{what} log p(z) at {it}")
        assert np.array_equal(a0, a1), f"{what}: decisions differ at {it}"
        fin = np.isfinite(l0)
        assert np.allclose(l1[fin], l0[fin], rtol=0, atol=1e-7 * max(1.0, np.abs(l0[fin]).max()))
        assert_close(x1, x0, 1e-9, f"{what} paths at {it}")


@pytest.mark.parametrize("d", [8, 40])
def test_l96_stencil_direct_matches_generic(mods, d):
    """The DMMA panel elimination (d <= 43)."""
    _, auxk, bm = mods
    T = 64
    spec = bm.ModelSpec(kind="lorenz96", T=T, dx=d, data_seed=3)
    lat, data = bm.simulate(spec)
    tg = auxk.make_target(spec, data)
    assert tg.exact_sel == 1 and tg.q == (d + 1) // 2
    gen, fused = _pair(mods, tg, lat, 0.05, 4, 4)
    _compare(gen, fused, f"L96 d={d}")


def test_rank1_form_matches_generic(mods):
    """d = 49 (spatio-temporal grid 7, no exact rows): past the DMMA panel form's d <= 43,
    the rank-1 register-tile elimination."""
    _, auxk, bm = mods
    T = 24
    spec = bm.ModelSpec(kind="spatio-temporal", T=T, grid=7, data_seed=5)
    lat, data = bm.simulate(spec)
    tg = auxk.make_target(spec, data)
    assert tg.dx == 49 and tg.exact_sel == 1
    gen, fused = _pair(mods, tg, lat, 0.5, 2, 2)
    _compare(gen, fused, "spatio d=49")


def test_l96_partial_exact_blocks(mods):
    """emask mixed (exact_tv): steps without the exact block keep the generic model's
    N(0; 0, 1) rows (k_build_HR) in log p(z)."""
    _, auxk, bm = mods
    T, d = 48, 12
    spec = bm.ModelSpec(kind="lorenz96", T=T, dx=d, data_seed=4)
    lat, data = bm.simulate(spec)
    tg = auxk.make_target(spec, data)
    em = np.ones(T + 1, np.uint8)
    em[5:11] = 0
    em[30] = 0
    tg.emask = torch.as_tensor(em, device=tg.device)
    tg.emask_host = em
    tg.exact_tv = 1
    gen, fused = _pair(mods, tg, lat, 0.05, 4, 3)
    _compare(gen, fused, "L96 mixed emask")


@pytest.mark.parametrize("kind,kw", [("stochvol", dict(dx=3)), ("spatio-temporal", dict(grid=3))])
def test_linear_targets_dense_direct_matches_generic(mods, kind, kw):
    _, auxk, bm = mods
    T = 40
    spec = bm.ModelSpec(kind=kind, T=T, data_seed=11, **kw)
    lat, data = bm.simulate(spec)
    tg = auxk.make_target(spec, data)
    assert tg.exact_sel == 1
    for backend in (0, 1):
        gen, fused = _pair(mods, tg, lat, 0.5, 3, 3, backend)
        _compare(gen, fused, f"{kind} backend {backend}")


def test_broken_structure_contract_aborts(mods):
    """exact_sel set on a target whose exact rows are not unit selections: the fused
    filter refuses (status 3) and the step is an abort, never a silent wrong answer."""
    _lib, auxk, bm = mods
    T = 16
    spec = bm.ModelSpec(kind="lgssm-synthetic", T=T, dx=3, dy=2, data_seed=2)
    lat, data = bm.simulate(spec)
    tg = auxk.make_target(spec, data)
    assert tg.exact_sel == 0  # dense H
    ok = auxk.init_chains(tg, lat, 0.5, 5, 2)
    ok.kernel_step(0)
    assert int(ok.aborted.sum()) == 0
    tg.exact_sel = 1
    bad = auxk.init_chains(tg, lat, 0.5, 5, 2)
    bad.kernel_step(0)
    assert int(bad.aborted.sum()) == 2
