"""Pins the C restatement (oracle/, the checker every GPU test uses) to the REFERENCE
ITSELF: oracle/_ref is /root/reference/proj/src compiled unmodified against the Eigen /
doctest shims (oracle/ref.mk), driven through oracle/ref_bridge.cpp (CPU only).

Bars (BASELINE.json north_star): integer / key / index / accept decisions bit-exact
outside the near-tie band; paths, moments, log-likelihoods and log alpha within 1e-12
relative (the two sides differ only in the LLT / triangular-solve rounding of the
Eigen stand-in vs the restatement, ~1e-15).  Near ties: a decision whose margin
|ln U - log alpha| (or a cSMC cumulative-weight margin) is below the band
T * 64 * eps * (scale of the summed terms) may legitimately differ; the tests count
them, require identical decisions outside the band, and stop comparing a chain after
a tie flip (its states diverge from there on).
"""
import json
import math
import os
import pathlib
import subprocess

import numpy as np
import pytest

from oracle import pyoracle as O
from testutil import random_model, simulate_obs

R = pytest.importorskip("oracle.refbridge")
EPS = np.finfo(np.float64).eps


@pytest.fixture(scope="module", autouse=True)
def _ref_built():
    O.build()
    if not R.available():
        try:
            R.build()
        except RuntimeError as e:
            pytest.skip(f"oracle/_ref not built and not buildable here: {e}")


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b))))


def tie_band(T, scale):
    """Rounding band of a sum of ~T terms of magnitude `scale`."""
    return max(T, 1) * 64 * EPS * max(1.0, abs(scale))


# ---------------------------------------------------------------- RNG (rng.hpp)
def test_rng_keys_and_draws_bit_exact():
    """rng.hpp:35-118: keys, uniforms, normals, next_key — port == reference bit for bit."""
    for seed in (0, 1, 7, 2 ** 63 + 5):
        root = O.from_seed(seed)
        assert R.from_seed_key(seed) == root.key
        for label, index in ((1, 0), (7, 3), (12, 65535), (15, 2 ** 40)):
            s = O.derive(root, label, index)
            assert R.derive_key(root.key, label, index) == s.key
            n = O.normal_vec(O.derive(root, label, index), 32)
            assert np.array_equal(R.draws(s.key, "normal", 32), n)
            s2 = O.derive(root, label, index)
            u = np.array([O.next_uniform(s2) for _ in range(16)])
            assert np.array_equal(R.draws(s.key, "uniform", 16), u)


# ---------------------------------------------------------------- models (models.cpp)
KINDS = [("lgssm-synthetic", dict(T=60, dx=4, dy=2, data_seed=3)),
         ("lgssm-synthetic", dict(T=40, dx=1, dy=1, data_seed=1)),
         ("stochvol", dict(T=50, dx=3, data_seed=11)),
         ("diffusion-smoothing", dict(T=40)),
         ("spatio-temporal", dict(T=30, grid=3, data_seed=7)),
         ("spatio-temporal", dict(T=20, grid=4, data_seed=7)),
         ("grid-1d-test", dict(T=30))]


@pytest.mark.parametrize("kind,kw", KINDS)
def test_simulate_and_target_match_reference(kind, kw):
    """models.cpp:162-336: simulated latents/data, log_gamma and potential gradients."""
    s = O.spec(kind, **kw)
    lo, do = O.simulate(s)
    lr, dr = R.simulate(s)
    assert rel(lo, lr) < 1e-12
    if kind == "spatio-temporal":  # Poisson counts: integers, exact
        assert np.array_equal(do, dr)
    else:
        assert rel(do, dr) < 1e-12
    to, tr = O.make_target(s, dr), R.make_target(s, dr)
    assert rel(to.log_gamma(lr), tr.log_gamma(lr)) < 1e-12
    for t in (0, s.T // 2, s.T):
        assert rel(to.grad_pot(t, lr[t]), tr.grad_pot(t, lr[t])) < 1e-12
        assert rel(to.log_pot(t, lr[t]), tr.log_pot(t, lr[t])) < 1e-12


def test_lorenz96_target_matches_reference_tractable_target():
    """The L96 target (C3) on the reference's GenSSMTarget::tractable (target.cpp:29-45)."""
    s = O.spec("lorenz96", T=30, dx=40, data_seed=3)
    lat, data = O.simulate(s)
    to, tr = O.make_target(s, data), R.make_target(s, data)
    assert rel(to.log_gamma(lat), tr.log_gamma(lat)) < 1e-12
    for t in (0, 17, 30):
        assert rel(to.grad_pot(t, lat[t]), tr.grad_pot(t, lat[t])) < 1e-12


# ---------------------------------------------------------------- LGSSM + samplers
MODELS = [(5, 1, 1, False, False), (40, 4, 2, False, False), (33, 3, 2, True, True),
          (24, 9, 5, True, False), (12, 16, 3, False, True)]


@pytest.mark.parametrize("T,dx,dy,tv,mask", MODELS)
def test_filters_samplers_logpdf_match_reference(T, dx, dy, tv, mask):
    """lgssm.cpp:73-199, pit.cpp:78-301: both filters, the three samplers (stream and
    pre-drawn noise) and path_logpdf on random models (testutil.hpp:35-68)."""
    s = O.derive(O.from_seed(100 + T), O.L_SIMULATE, dx)
    m = random_model(s, T, dx, dy, time_varying=tv, with_mask=mask)
    obs = simulate_obs(m, O.from_seed(200 + dx))
    rm = R.RModel(m)
    fo, fr = O.kalman_filter(m, obs), R.kalman_filter(rm, obs)
    for a in ("pred_mean", "pred_cov", "filt_mean", "filt_cov"):
        assert rel(getattr(fo, a), getattr(fr, a)) < 1e-12, a
    assert rel(fo.log_marginal, fr.log_marginal) < 1e-12
    po, _ = O.parallel_filter(m, obs)
    pr = R.parallel_filter(rm, obs)
    assert rel(po.filt_mean, pr.filt_mean) < 1e-11
    assert rel(po.filt_cov, pr.filt_cov) < 1e-11
    assert rel(po.log_marginal, pr.log_marginal) < 1e-12
    rng = np.random.default_rng(T * 31 + dx)
    n_nodes = 2 * T + 2
    pre = dict(terminal=rng.standard_normal(dx), backward=rng.standard_normal((T, dx)),
               bridge=rng.standard_normal((n_nodes * 2, dx)))
    root = O.derive(O.from_seed(1), O.L_CHAIN, 5)
    for name in ("backward_sample", "prefix_sample", "dnc_sample"):
        xo = getattr(O, name)(m, fo, O.stream_noise(root))
        xr = getattr(R, name)(rm, fr, root)
        assert rel(xo, xr) < 1e-11, name
        nz, keep = O.predrawn_noise(dx, pre["terminal"], pre["backward"], pre["bridge"])
        xo = getattr(O, name)(m, fo, nz)
        xr = getattr(R, name)(rm, fr, pre)
        assert rel(xo, xr) < 1e-11, name + " predrawn"
        assert rel(O.path_logpdf(m, obs, xo, fo), R.path_logpdf(rm, obs, xr, fr)) < 1e-12


# ---------------------------------------------------------------- aux Kalman (auxk.cpp)
def run_aux_pair(s, iters, backend, parallel, zeroth=False, delta=None, adapt=None):
    lat, data = O.simulate(s) if s.kind == O.KIND["lorenz96"] else R.simulate(s)
    to, tr = O.make_target(s, data), R.make_target(s, data)
    x0 = np.repeat(to.arrays()["m0"][None, :] if hasattr(to, "arrays") else lat[:1], s.T + 1, 0)
    d0 = delta if delta is not None else 1.0
    co, cr = O.AuxChain(to, x0, d0), R.AuxChain(tr, x0, d0)
    root = O.derive(O.from_seed(1), O.L_CHAIN, 0)
    flips = compared = 0
    for it in range(iters):
        co.step(root, backend, int(parallel), int(zeroth))
        cr.step(root, backend, parallel, zeroth)
        so, sr = co.c.stats, cr.state()
        la_o, la_r = so.last_log_alpha, sr["last_log_alpha"]
        if so.accepted != sr["accepted"] or so.aborted != sr["aborted"]:
            # the decision differs: legitimate only inside the near-tie band
            u = O.next_uniform(O.derive(O.derive(root, O.L_ITERATION, it), O.L_MH_ACCEPT, 0))
            margin = abs(math.log(u) - la_r)
            band = tie_band(s.T * O.latent_dim(s), sr["log_gamma"])
            assert margin <= band, f"iteration {it}: decision differs outside the tie band " \
                                   f"(margin {margin:.3e} > band {band:.3e})"
            flips += 1
            break
        compared += 1
        if math.isfinite(la_r):
            assert abs(la_o - la_r) <= 1e-9 * max(1.0, abs(la_r)), f"log alpha at {it}"
        assert rel(co.x, sr["x"]) < 1e-9, f"path at {it}"
        assert rel(co.c.delta, sr["delta"]) < 1e-10  # exp(log alpha) enters the update
        if adapt is not None:
            co.adapt(adapt)
            cr.adapt(adapt)
    return compared, flips, cr.state()


AUX_CASES = [
    # C1 (configs[0]) at its own size: 1-D LGSSM, T = 1024, prefix backend
    ("c1-prefix", O.spec("lgssm-synthetic", T=1024, dx=1, dy=1, data_seed=1), 12, 1, False),
    ("c1-prefix-scan", O.spec("lgssm-synthetic", T=1024, dx=1, dy=1, data_seed=1), 6, 1, True),
    ("lgssm-seq", O.spec("lgssm-synthetic", T=80, dx=3, dy=2, data_seed=5), 8, 0, False),
    ("lgssm-dnc", O.spec("lgssm-synthetic", T=80, dx=3, dy=2, data_seed=5), 8, 2, False),
    ("stochvol", O.spec("stochvol", T=120, dx=3, data_seed=11), 10, 1, False),
    ("stochvol-seq-scan", O.spec("stochvol", T=60, dx=3, data_seed=11), 8, 0, True),
    ("l63", O.spec("diffusion-smoothing", T=80), 8, 1, False),
    # C5 model at reduced T (d = 16), scan filter as the config runs it
    ("c5-spatio", O.spec("spatio-temporal", T=64, grid=4, data_seed=7), 4, 1, True),
    ("spatio9-dnc", O.spec("spatio-temporal", T=48, grid=3, data_seed=7), 6, 2, False),
    ("grid1d", O.spec("grid-1d-test", T=40), 10, 0, False),
]


@pytest.mark.parametrize("name,s,iters,backend,parallel", AUX_CASES, ids=[c[0] for c in AUX_CASES])
def test_aux_kernel_step_matches_reference(name, s, iters, backend, parallel):
    """auxk.cpp:130-198 chained over iterations with burn-in adaptation (auxk.cpp:213-218):
    accept decisions identical, log alpha / paths / delta within tolerance."""
    compared, flips, st = run_aux_pair(s, iters, backend, parallel, adapt=0.574)
    assert compared + flips == iters or flips == 1
    assert st["iter"] == compared + flips


def test_aux_zeroth_order_and_c3_l96_match_reference():
    """zeroth_order (auxk.cpp:97-101) and the C3 model (L96, d = 40) at reduced T."""
    s = O.spec("stochvol", T=50, dx=3, data_seed=11)
    run_aux_pair(s, 6, 1, False, zeroth=True)
    s = O.spec("lorenz96", T=16, dx=40, data_seed=3)
    compared, flips, _ = run_aux_pair(s, 2, 0, False, delta=0.05)
    assert compared + flips == 2


def test_mh_log_ratio_matches_reference():
    """auxk.cpp:200-211 and sample_aux_obs (:45-54)."""
    s = O.spec("stochvol", T=40, dx=3, data_seed=11)
    lat, data = R.simulate(s)
    to, tr = O.make_target(s, data), R.make_target(s, data)
    it = O.derive(O.derive(O.from_seed(3), O.L_CHAIN, 0), O.L_ITERATION, 0)
    uo, ur = O.sample_aux_obs(lat, 0.7, it), R.sample_aux_obs(lat, 0.7, it)
    assert np.array_equal(uo, ur)
    xp = lat + 0.05
    assert rel(O.mh_log_ratio(to, lat, xp, uo, 0.7), R.mh_log_ratio(tr, lat, xp, ur, 0.7)) < 1e-11


# ---------------------------------------------------------------- particle Gibbs (fkpg.cpp)
@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("N", [8, 64, 256])
def test_pgibbs_matches_reference(mode, N):
    """aux_pgibbs_step (fkpg.cpp:252-271) over a few iterations on stochvol (C4's model
    at reduced T): reference paths, keys and update flags identical; the first step's
    ancestors and backward indices identical (csmc_step, fkpg.cpp:112-152)."""
    T = 40 if N == 256 else 60
    s = O.spec("stochvol", T=T, dx=3, data_seed=11)
    lat, data = R.simulate(s)
    to, tr = O.make_target(s, data), R.make_target(s, data)
    x0 = np.tile(np.full(3, s.sv_mu), (T + 1, 1))
    po, pr = O.PGChain(to, x0, 1.0), R.PGChain(tr, x0, 1.0)
    root = O.derive(O.from_seed(1), O.L_CHAIN, 0)
    # first step, index level
    it = O.derive(root, O.L_ITERATION, 0)
    u = R.sample_aux_obs(x0, 1.0, it)
    st_r, bad_r, anc_r, traj_r = R.csmc_trace(tr, x0, np.zeros(T + 1, np.uint64), u, 1.0, N, it, mode)
    st_o, bad_o, anc_o, sel_o = po.step(N, root, mode=mode, trace=True)
    assert st_r == 0 and st_o == 0
    assert np.array_equal(anc_o[1:], anc_r[1:]), "ancestor indices"
    assert rel(po.x, traj_r) == 0.0 or rel(po.x, traj_r) < 1e-12
    pr.step(N, root, mode=mode)
    for k in range(1, 4):
        po.step(N, root, mode=mode)
        pr.step(N, root, mode=mode)
        sr = pr.state()
        assert np.array_equal(po.keys, sr["keys"]), f"keys at iteration {k}"
        assert rel(po.x, sr["x"]) < 1e-12, f"path at iteration {k}"
        assert po.p.updates == sr["updates"]
        po.adapt(0.9)
        pr.adapt(0.9)
        assert rel(po.p.delta, pr.state()["delta"]) < 1e-14


# ---------------------------------------------------------------- the reference's own suites
def test_reference_unit_suite_runs_green_on_the_shim():
    """proj/tests/test_*.cpp compiled unmodified against the shims: a fast subset here
    (known answers, jitter ladder, scan trees, bit-equalities, exact acceptance, the
    failure paths); the full 115-case suite and acceptance.cpp are recorded in
    profiles/r2_ref/ (`oracle/_ref/auxmc_tests`, `oracle/_ref/acceptance`)."""
    exe = pathlib.Path(R.REF_DIR) / "auxmc_tests"
    if not exe.exists():
        pytest.skip("oracle/_ref/auxmc_tests not built")
    for sel in ("stream", "log_pdf", "jitter", "scan", "realize_noise", "horizon one",
                "exactly representable", "antisymmetric", "collapsed weights", "brute-force",
                "outside the support", "non-finite proposal"):
        r = subprocess.run([str(exe), f"-tc={sel}"], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stdout + r.stderr
