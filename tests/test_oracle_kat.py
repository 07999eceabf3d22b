"""Pins the CPU oracle to the reference's own known answers (CPU only).

Each test restates a check from proj/tests/*.cpp (file:line in the docstring)
against oracle/ (the checker every GPU parity test relies on).
"""
import math

import numpy as np
import pytest

from testutil import random_model, random_spd, simulate_obs

LOG2PI = 1.8378770664093454835606594728112


# ---------------------------------------------------------------- rng (test_rng.cpp)
def test_rng_replay_and_interleaving(oracle):
    """test_rng.cpp:11-40: a stream is a pure function of its path."""
    a = oracle.derive(oracle.from_seed(5), 3, 7)
    b = oracle.derive(oracle.from_seed(5), 3, 7)
    xa = [oracle.next_normal(a) for _ in range(5)]
    _ = oracle.derive(oracle.from_seed(5), 4, 1)  # unrelated stream in between
    xb = [oracle.next_normal(b) for _ in range(5)]
    assert xa == xb


def test_rng_distinct_keys_for_label_index_paths(oracle):
    """test_rng.cpp:42-58: 15 labels × 16 indices give distinct keys."""
    root = oracle.from_seed(1)
    keys = {oracle.derive(root, l, i).key for l in range(1, 16) for i in range(16)}
    assert len(keys) == 15 * 16


def test_rng_uniform_open_interval_and_moments(oracle):
    """test_rng.cpp:60-90: uniforms in (0,1); normal mean ~0, var ~1."""
    s = oracle.derive(oracle.from_seed(9), oracle.L_SIMULATE, 0)
    u = np.array([oracle.next_uniform(s) for _ in range(20000)])
    assert u.min() > 0.0 and u.max() < 1.0
    s = oracle.derive(oracle.from_seed(9), oracle.L_SIMULATE, 1)
    z = oracle.normal_vec(s, 20000)
    assert abs(z.mean()) < 4 / math.sqrt(20000)
    assert abs(z.var() - 1.0) < 4 * math.sqrt(2 / 20000)


def test_rng_normal_vec_equals_next_normal(oracle):
    """test_rng.cpp:92-100"""
    a = oracle.derive(oracle.from_seed(3), 1, 2)
    b = oracle.derive(oracle.from_seed(3), 1, 2)
    v = oracle.normal_vec(a, 6)
    w = np.array([oracle.next_normal(b) for _ in range(6)])
    assert np.array_equal(v, w)


def test_host_rng_matches_product_library(oracle):
    """The product's host RNG (libauxmc_b200) is bit-exact with the oracle."""
    from paper_2303_00301_b200 import rng
    for seed in (0, 1, 7, 2 ** 63 + 5):
        for label, index in ((1, 0), (7, 3), (15, 99999)):
            want = oracle.derive(oracle.from_seed(seed), label, index)
            got = rng.RngStream.from_seed(seed).derive(label, index)
            assert got.key == want.key
            assert [got.next_normal() for _ in range(3)] == [oracle.next_normal(want) for _ in range(3)]
            assert got.next_uniform() == oracle.next_uniform(want)


# ---------------------------------------------------------------- gauss (test_gauss.cpp)
def test_log_pdf_closed_forms(oracle):
    """test_gauss.cpp:15-31"""
    assert abs(oracle.log_pdf([0.0], [0.0], [[1.0]]) - (-0.9189385332046727)) < 1e-12
    for d in (1, 2, 5):
        m = np.full(d, 0.7)
        assert abs(oracle.log_pdf(m, m, np.eye(d)) - (-0.5 * d * LOG2PI)) < 1e-12
    want = -0.5 * math.log(2 * math.pi * 4.0) - 1.0 / 8.0
    assert abs(oracle.log_pdf([1.0], [0.0], [[4.0]]) - want) < 1e-12


def test_chol_psd_jitter_policy(oracle):
    """test_gauss.cpp:161-173: near-singular admitted, zero -> zero, negative fails."""
    a = np.ones((3, 3))
    a[2, 2] += 1e-13
    l = oracle.chol_psd(a)
    assert np.max(np.abs(l @ l.T - a)) < 1e-8
    assert np.all(oracle.chol_psd(np.zeros((2, 2))) == 0.0)
    with pytest.raises(RuntimeError):
        oracle.chol_psd(-np.eye(2))


def test_spectral_radius(oracle):
    """models.cpp:58 uses |eig|max; compare with LAPACK."""
    g = np.random.default_rng(0)
    for n in (1, 2, 3, 4, 7, 16, 40):
        a = g.standard_normal((n, n))
        assert abs(oracle.spectral_radius(a) - np.max(np.abs(np.linalg.eigvals(a)))) < 1e-10 * n


# ---------------------------------------------------------------- lgssm (test_lgssm.cpp)
def scalar_model(oracle, T, m0, p0, f, b, q, h, c, r, mask=None):
    return oracle.Model.homogeneous(T, [m0], [[p0]], [[f]], [b], [[q]], [[h]], [c], [[r]], mask)


def test_filter_scalar_posterior_halves_variance(oracle):
    """test_lgssm.cpp:43-55"""
    m = scalar_model(oracle, 0, 0.0, 1.0, 1.0, 0.0, 1.0, 1.0, 0.0, 1.0)
    fr = oracle.kalman_filter(m, np.zeros((1, 1)))
    assert abs(fr.filt_mean[0, 0]) < 1e-12
    assert abs(fr.filt_cov[0, 0, 0] - 0.5) < 1e-12
    assert abs(fr.log_marginal - oracle.log_pdf([0.0], [0.0], [[2.0]])) < 1e-12


def test_filter_fully_masked_is_prior_propagation(oracle):
    """test_lgssm.cpp:57-90"""
    T = 6
    s = oracle.derive(oracle.from_seed(4), oracle.L_SIMULATE, 0)
    base = random_model(s, T, 2, 1)
    m = oracle.Model(T, base.m0, base.P0, base.F, base.b, base.Q, base.H, base.c, base.R,
                     np.zeros(T + 1, np.uint8))
    fr = oracle.kalman_filter(m, np.zeros((T + 1, 1)))
    assert fr.log_marginal == 0.0
    mean, cov = m.m0.copy(), m.P0.copy()
    for t in range(T + 1):
        if t > 0:
            mean = m.F[0] @ mean + m.b[0]
            cov = m.F[0] @ cov @ m.F[0].T + m.Q[0]
        assert np.max(np.abs(fr.filt_mean[t] - mean)) < 1e-12
        assert np.max(np.abs(fr.filt_cov[t] - cov)) < 1e-10


@pytest.mark.parametrize("seed", range(1, 11))
def test_filter_and_smoother_match_dense_oracle(oracle, seed):
    """test_lgssm.cpp:92-112, :350-383: filter evidence and smoother vs dense."""
    s = oracle.derive(oracle.from_seed(seed), oracle.L_SIMULATE, 5)
    m = random_model(s, 2 + seed % 6, 1 + seed % 3, 1 + seed % 2, seed % 2 == 0, seed % 3 == 0)
    obs = simulate_obs(m, oracle.from_seed(50 + seed))
    fr = oracle.kalman_filter(m, obs)
    mean, cov, le = oracle.dense_oracle(m, obs)
    assert abs(fr.log_marginal - le) < 1e-8
    sm, sc = oracle.rts_smoother(m, fr)
    d = m.dx
    for t in range(m.T + 1):
        assert np.max(np.abs(sm[t] - mean[t * d:(t + 1) * d])) < 1e-7
        assert np.max(np.abs(sc[t] - cov[t * d:(t + 1) * d, t * d:(t + 1) * d])) < 1e-7


def test_dense_oracle_two_step_scalar(oracle):
    """test_lgssm.cpp:324-341: hand-conditioned two-step scalar case."""
    p0, f, q, r, y1 = 1.0, 0.5, 0.3, 0.4, 0.8
    m = scalar_model(oracle, 1, 0.0, p0, f, 0.0, q, 1.0, 0.0, r, np.array([0, 1], np.uint8))
    mean, cov, _ = oracle.dense_oracle(m, np.array([[0.0], [y1]]))
    joint = np.array([[p0, f * p0], [f * p0, f * f * p0 + q]])
    s = joint[1, 1] + r
    want_mean = np.array([joint[0, 1] / s * y1, joint[1, 1] / s * y1])
    want_cov = joint - np.outer(joint[:, 1], joint[:, 1]) / s
    assert np.max(np.abs(mean - want_mean)) < 1e-12
    assert np.max(np.abs(cov - want_cov)) < 1e-12


def test_backward_elements_limits(oracle):
    """test_pit.cpp:58-84: uninformative future collapses to the filtered law;
    deterministic copy dynamics give identity maps."""
    T = 3
    m = scalar_model(oracle, T, 0.2, 1.0, 0.9, 0.0, 1e12, 1.0, 0.0, 0.5)
    fr = oracle.kalman_filter(m, np.array([[0.1], [-0.4], [0.3], [0.2]]))
    for t in range(T):
        G, off, cov = oracle.backward_step(m, fr, t)
        assert abs(G[0, 0]) < 1e-9
        assert abs(off[0] - fr.filt_mean[t, 0]) <= 1e-6 * abs(fr.filt_mean[t, 0]) + 1e-12
        assert abs(cov[0, 0] - fr.filt_cov[t, 0, 0]) <= 1e-6 * fr.filt_cov[t, 0, 0]
    T = 4
    m = scalar_model(oracle, T, 0.0, 1.0, 1.0, 0.0, 0.0, 1.0, 0.0, 0.5)
    fr = oracle.kalman_filter(m, np.zeros((T + 1, 1)))
    for t in range(T):
        G, off, cov = oracle.backward_step(m, fr, t)
        assert abs(G[0, 0] - 1.0) < 1e-10 and abs(off[0]) < 1e-10 and abs(cov[0, 0]) < 1e-10


def test_aux_model_scalar_conjugate_posterior(oracle):
    """test_target_auxk.cpp:153-180: exact potential + aux row == conjugate update."""
    m0, p0, r, y, uu, delta = 0.3, 1.2, 0.5, 0.9, -0.1, 0.8
    m = scalar_model(oracle, 0, m0, p0, 1.0, 0.0, 1.0, 1.0, 0.0, r)
    tg = oracle.target_from_lgssm(m, np.array([[y]]), generic=False)
    fr, obs = oracle.aux_model_filter(tg, np.array([[0.2]]), np.array([[uu]]), delta)
    prec = 1.0 / p0 + 1.0 / r + 2.0 / delta
    mean = (m0 / p0 + y / r + 2.0 * uu / delta) / prec
    assert abs(fr.filt_mean[0, 0] - mean) < 1e-10 * abs(mean)
    assert abs(fr.filt_cov[0, 0, 0] - 1.0 / prec) < 1e-10 / prec


def test_aux_model_potential_free_observes_noisy_copies(oracle):
    """test_target_auxk.cpp:119-134: z = u, H = 1, R = δ/2 with no potentials."""
    T = 3
    m = scalar_model(oracle, T, 0.0, 1.0, 0.9, 0.0, 0.2, 1.0, 0.0, 1.0,
                     np.zeros(T + 1, np.uint8))
    tg = oracle.target_from_lgssm(m, np.zeros((T + 1, 1)), generic=False)
    u = np.array([[0.1], [-0.2], [0.3], [0.0]])
    fr, obs = oracle.aux_model_filter(tg, np.zeros((T + 1, 1)), u, 0.5)
    assert np.array_equal(obs[:, :1], u)
    # posterior of a 0.9-AR(1) observed through z = u with variance 0.25
    want = oracle.kalman_filter(oracle.Model.homogeneous(T, [0.0], [[1.0]], [[0.9]], [0.0], [[0.2]],
                                                         [[1.0]], [0.0], [[0.25]]), u)
    assert np.max(np.abs(fr.filt_mean - want.filt_mean)) < 1e-12


# ---------------------------------------------------------------- pit (test_pit.cpp)
@pytest.mark.parametrize("seed", range(1, 11))
def test_sampler_laws_equal_dense_posterior(oracle, seed):
    """test_pit.cpp:283-337, runner.cpp:279-298: exact affine law of all three
    samplers equals dense conditioning (< 1e-8)."""
    from oracle import pyoracle as O
    s = O.spec("lgssm-synthetic", T=2 + seed % 5, dx=1 + seed % 3, dy=1 + (seed // 2) % 2,
               data_seed=seed)
    lat, data = O.simulate(s)
    m = O.synthetic_lgssm(s)
    fr = O.kalman_filter(m, data)
    mean, cov, _ = O.dense_oracle(m, data)
    for which in range(3):
        lm, lc = O.extract_affine_law(which, m, fr)
        assert max(np.max(np.abs(lm - mean)), np.max(np.abs(lc - cov))) < 1e-8


def test_prefix_agrees_with_sequential_on_shared_streams(oracle):
    """test_pit.cpp:136-148 (< 1e-8) and :150-159 (bit-equal at T = 1)."""
    s = oracle.derive(oracle.from_seed(8), oracle.L_SIMULATE, 3)
    m = random_model(s, 25, 2, 1)
    obs = simulate_obs(m, oracle.from_seed(81))
    fr = oracle.kalman_filter(m, obs)
    for i in range(25):
        key = oracle.derive(oracle.from_seed(200), oracle.L_CHAIN, i)
        seq = oracle.backward_sample(m, fr, oracle.stream_noise(key))
        par = oracle.prefix_sample(m, fr, oracle.stream_noise(key))
        assert np.max(np.abs(seq - par)) < 1e-8
    s = oracle.derive(oracle.from_seed(9), oracle.L_SIMULATE, 4)
    m = random_model(s, 1, 3, 2)
    obs = simulate_obs(m, oracle.from_seed(91))
    fr = oracle.kalman_filter(m, obs)
    key = oracle.from_seed(17)
    seq = oracle.backward_sample(m, fr, oracle.stream_noise(key))
    assert np.array_equal(seq, oracle.prefix_sample(m, fr, oracle.stream_noise(key)))
    assert np.array_equal(seq, oracle.dnc_sample(m, fr, oracle.stream_noise(key)))


def test_parallel_filter_agrees_with_kalman_filter(oracle):
    """test_pit.cpp:188-229"""
    s = oracle.derive(oracle.from_seed(10), oracle.L_SIMULATE, 6)
    for T, mask in ((0, False), (50, False), (40, True)):
        m = random_model(s, T, 2, 1, False, mask)
        obs = simulate_obs(m, oracle.from_seed(11 + T))
        a = oracle.kalman_filter(m, obs)
        b, _ = oracle.parallel_filter(m, obs)
        tol = 1e-12 if T == 0 else (1e-9 if mask else 1e-6)
        assert np.max(np.abs(a.filt_mean - b.filt_mean)) < tol
        assert np.max(np.abs(a.filt_cov - b.filt_cov)) < tol
        assert abs(a.log_marginal - b.log_marginal) < tol * max(1, abs(a.log_marginal))


def test_scan_span_is_ceil_log2(oracle):
    """test_scan.cpp:66-80, test_pit.cpp:366-378: Sklansky critical path."""
    s = oracle.derive(oracle.from_seed(12), oracle.L_SIMULATE, 7)
    for T in (1, 2, 5, 16, 33):
        m = random_model(s, T, 1, 1)
        obs = simulate_obs(m, oracle.from_seed(T))
        fr = oracle.kalman_filter(m, obs)
        _, (cp, apps) = oracle.prefix_sample(m, fr, oracle.stream_noise(oracle.from_seed(1)),
                                             stats=True)
        assert cp == (math.ceil(math.log2(T)) if T > 1 else 0)


# ---------------------------------------------------------------- auxk (test_target_auxk.cpp)
@pytest.mark.parametrize("backend", [0, 1, 2])
def test_exact_target_unit_acceptance(oracle, backend):
    """test_target_auxk.cpp:182-231, runner.cpp:300-313: |log α| < 1e-8."""
    s = oracle.spec("lgssm-synthetic", T=10, dx=2, dy=1, data_seed=3)
    lat, data = oracle.simulate(s)
    tg = oracle.make_target(s, data)
    ch = oracle.AuxChain(tg, np.tile(tg.arrays()["m0"], (11, 1)), 0.8)
    rng = oracle.from_seed(99)
    for _ in range(50):
        ch.step(rng, backend)
        assert abs(ch.c.stats.last_log_alpha) < 1e-8
    assert ch.c.stats.accepted == 50


def test_log_alpha_antisymmetry(oracle):
    """test_target_auxk.cpp:317-332"""
    so = oracle.spec("stochvol", T=20, dx=3, data_seed=11)
    lat, data = oracle.simulate(so)
    tg = oracle.make_target(so, data)
    x = lat
    xp = lat + 0.05 * np.sin(np.arange(lat.size)).reshape(lat.shape)
    u = x + 0.3
    a = oracle.mh_log_ratio(tg, x, xp, u, 0.6)
    b = oracle.mh_log_ratio(tg, xp, x, u, 0.6)
    assert abs(a + b) < 1e-9


@pytest.mark.parametrize("kind,kw", [("stochvol", dict(dx=3, data_seed=11)),
                                     ("spatio-temporal", dict(grid=3, data_seed=7)),
                                     ("diffusion-smoothing", dict(data_seed=3)),
                                     ("lorenz96", dict(dx=8, data_seed=3)),
                                     ("grid-1d-test", dict())])
def test_model_gradients_match_finite_differences(oracle, kind, kw):
    """test_bench.cpp:414-440: ∇ log g vs central differences (h = 1e-5 (1+|x|))."""
    so = oracle.spec(kind, T=4, **kw)
    lat, data = oracle.simulate(so)
    tg = oracle.make_target(so, data)
    for t in range(so.T + 1):
        x = lat[t]
        g = tg.grad_pot(t, x)
        fd = np.zeros_like(x)
        for i in range(x.size):
            h = 1e-5 * (1 + abs(x[i]))
            hi, lo = x.copy(), x.copy()
            hi[i] += h
            lo[i] -= h
            fd[i] = (tg.log_pot(t, hi) - tg.log_pot(t, lo)) / (2 * h)
        assert np.max(np.abs(g - fd)) < 1e-4 * max(1.0, np.max(np.abs(g)))


def test_bench_models_product_match_oracle(oracle):
    """Host-side product models (host/models.cpp) reproduce the oracle's data."""
    from paper_2303_00301_b200 import bench_models as bm
    for kind, kw in (("lgssm-synthetic", dict(dx=4, dy=1)), ("stochvol", dict(dx=3, data_seed=11)),
                     ("spatio-temporal", dict(grid=4, data_seed=7)),
                     ("diffusion-smoothing", dict(data_seed=3)), ("lorenz96", dict(dx=40, data_seed=3)),
                     ("grid-1d-test", dict())):
        a = bm.simulate(bm.ModelSpec(kind=kind, T=25, **kw))
        b = oracle.simulate(oracle.spec(kind, T=25, **kw))
        assert np.max(np.abs(a[0] - b[0])) < 1e-12
        if a[1].size:
            assert np.max(np.abs(a[1] - b[1])) < 1e-12


# ---------------------------------------------------------------- fkpg (test_fkpg.cpp)
def test_pgibbs_single_particle_keeps_reference(oracle):
    """test_fkpg.cpp:113-123: N = 1 returns the reference unchanged."""
    so = oracle.spec("stochvol", T=10, dx=3, data_seed=11)
    lat, data = oracle.simulate(so)
    tg = oracle.make_target(so, data)
    pg = oracle.PGChain(tg, lat, 1.0)
    pg.step(1, oracle.from_seed(1))
    assert np.array_equal(pg.x, lat)
    assert pg.p.updates == 0


@pytest.mark.parametrize("mode", [0, 1, 2])  # kPrior, kGradient, kFullyAdapted
def test_pgibbs_invariance_small_lgssm(oracle, mode):
    """runner.cpp:315-336 / acceptance.cpp:204-244: pgibbs moments agree with the
    dense posterior (|z| < 4.5) in every proposal mode."""
    s = oracle.spec("lgssm-synthetic", T=3, dx=1, dy=1, data_seed=11)
    lat, data = oracle.simulate(s)
    m = oracle.synthetic_lgssm(s)
    mean, cov, _ = oracle.dense_oracle(m, data)
    tg = oracle.make_target(s, data)
    pg = oracle.PGChain(tg, np.tile(tg.arrays()["m0"], (4, 1)), 1.0)
    rng = oracle.from_seed(7)
    draws = []
    for _ in range(3000):
        pg.step(8, rng, mode)
        draws.append(pg.x[:, 0].copy())
    draws = np.array(draws)
    # batch-means standard error
    nb = 30
    bm = draws[: (len(draws) // nb) * nb].reshape(nb, -1, 4).mean(axis=1)
    se = bm.std(axis=0, ddof=1) / np.sqrt(nb)
    z = np.abs(draws.mean(axis=0) - mean) / se
    assert np.all(z < 4.5), z


def test_grid_hmm_oracle_matches_dense_posterior(oracle):
    """grid_hmm.cpp:17-97 pinned on a 1-d linear Gaussian model, where the exact
    posterior is the dense conditioning one (midpoint-grid accuracy)."""
    s = oracle.spec("lgssm-synthetic", T=6, dx=1, dy=1, data_seed=4)
    lat, data = oracle.simulate(s)
    m = oracle.synthetic_lgssm(s)
    mean, cov, le = oracle.dense_oracle(m, data)
    tg = oracle.make_target(s, data)
    _, marg, gmean, gvar, gle = oracle.grid_hmm_posterior(tg, -8.0, 8.0, 1600)
    assert np.allclose(marg.sum(axis=1), 1.0)
    assert np.max(np.abs(gmean - mean)) < 1e-4
    assert np.max(np.abs(gvar - np.diag(cov))) < 1e-4
    assert abs(gle - le) < 1e-4
