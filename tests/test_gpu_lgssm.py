"""GPU parity: Kalman filter, pathwise samplers and path density vs the oracle.

Mirrors proj/tests/test_lgssm.cpp and test_pit.cpp: same-noise pathwise
agreement (test_pit.cpp:136-159), filter agreement (:188-229), masked steps
(test_lgssm.cpp:57-90), deterministic dynamics (test_pit.cpp:242-250), plus
the C2 shape class (one shared filter, many chains) at reduced horizon.
Tolerance: FP64 relative 1e-9 (BASELINE.json north_star).
"""
import numpy as np
import pytest
import torch

from conftest import assert_close
from testutil import predrawn, random_model, simulate_obs, to_gpu_model

pytestmark = pytest.mark.gpu

RTOL = 1e-9


@pytest.fixture(scope="module")
def gpu():
    from paper_2303_00301_b200 import _lib, lgssm, pit, rng
    assert _lib.load().auxmc_device_ok() == 1, "libauxmc_b200 sees no sm_100 device"
    return lgssm, pit, rng


CASES = [  # (T, dx, dy, time_varying, with_mask, seed)
    (9, 2, 1, False, False, 1),
    (25, 2, 1, True, False, 2),
    (40, 3, 2, True, True, 3),
    (1, 3, 2, False, False, 4),
    (0, 2, 1, False, False, 5),
    (129, 4, 1, False, False, 6),
    (300, 4, 2, True, True, 7),
    (50, 1, 1, False, True, 8),
    (64, 5, 3, False, False, 9),
]


def _oracle_case(oracle, T, dx, dy, tv, mask, seed):
    s = oracle.derive(oracle.from_seed(seed), oracle.L_SIMULATE, 1)
    m = random_model(s, T, dx, dy, tv, mask)
    obs = simulate_obs(m, oracle.from_seed(100 + seed))
    return m, obs


@pytest.mark.parametrize("case", CASES)
def test_kalman_filter_matches_oracle(gpu, oracle, case):
    lgssm, _, _ = gpu
    m, obs = _oracle_case(oracle, *case)
    want = oracle.kalman_filter(m, obs)
    fr = lgssm.kalman_filter(to_gpu_model(m), obs)
    assert int(fr.status[0]) == 0
    assert_close(fr.pred_mean[0].cpu(), want.pred_mean, RTOL, "pred_mean")
    assert_close(fr.pred_cov[0].cpu(), want.pred_cov, RTOL, "pred_cov")
    assert_close(fr.filt_mean[0].cpu(), want.filt_mean, RTOL, "filt_mean")
    assert_close(fr.filt_cov[0].cpu(), want.filt_cov, RTOL, "filt_cov")
    assert_close(fr.log_marginal[0].cpu(), want.log_marginal, RTOL, "log_marginal")


# CTA-group kernels (dims > 16): blocked LLT / triangular solves with DMMA
# panel updates, odd sizes to exercise partial 8-wide blocks and tiles.
LARGE_CASES = [
    (6, 20, 17, True, True, 31),
    (4, 17, 40, False, False, 32),
    (3, 40, 60, True, False, 33),
    (100, 10, 3, True, True, 34),   # warp groups; several prefix blocks
    (33, 12, 12, False, False, 35),
    (0, 10, 2, False, False, 39),   # edge horizons on the generic kernels
    (1, 12, 3, True, False, 40),
    (2, 9, 9, True, True, 41),
]


@pytest.mark.parametrize("case", LARGE_CASES)
def test_kalman_filter_large_dims_match_oracle(gpu, oracle, case):
    lgssm, _, _ = gpu
    m, obs = _oracle_case(oracle, *case)
    want = oracle.kalman_filter(m, obs)
    fr = lgssm.kalman_filter(to_gpu_model(m), obs)
    assert int(fr.status[0]) == 0
    assert_close(fr.pred_cov[0].cpu(), want.pred_cov, RTOL, "pred_cov")
    assert_close(fr.filt_mean[0].cpu(), want.filt_mean, RTOL, "filt_mean")
    assert_close(fr.filt_cov[0].cpu(), want.filt_cov, RTOL, "filt_cov")
    assert_close(fr.log_marginal[0].cpu(), want.log_marginal, RTOL, "log_marginal")


@pytest.mark.parametrize("sampler", [0, 1, 2])
@pytest.mark.parametrize("case", LARGE_CASES)
def test_samplers_large_dims_match_oracle(gpu, oracle, case, sampler):
    """d > 8: sequential (warp per path), generic blocked prefix scan, and the
    group DnC (CTA bridges for d > 16)."""
    lgssm, pit, _ = gpu

    m, obs = _oracle_case(oracle, *case)
    fr_o = oracle.kalman_filter(m, obs)
    gm = to_gpu_model(m)
    fr = lgssm.kalman_filter(gm, obs)
    B = 3
    term, back, bridge = predrawn(np.random.default_rng(case[-1]), B, m.T, m.dx,
                                  pit.dnc_bridge_count(m.T))
    want = _oracle_paths(oracle, sampler, m, fr_o, term, back, bridge)
    got = lgssm.PathSampler(gm, B, sampler, True)(fr, lgssm.Noise.predrawn(term, back, bridge))
    assert_close(got.cpu(), want, RTOL, f"sampler {sampler}")


@pytest.mark.parametrize("sampler", [0, 1, 2])
def test_samplers_d64_match_oracle(gpu, oracle, sampler):
    """d = 64: the backward elements' five-buffer and the DnC bridges' six-buffer
    CTA layouts fit where the eight-buffer ones exceeded shared memory;
    sequential, blocked prefix and DnC samplers against the oracle."""
    lgssm, pit, _ = gpu
    m, obs = _oracle_case(oracle, 5, 64, 8, True, False, 42)
    fr_o = oracle.kalman_filter(m, obs)
    gm = to_gpu_model(m)
    fr = lgssm.kalman_filter(gm, obs)
    assert int(fr.status[0]) == 0
    B = 2
    term, back, bridge = predrawn(np.random.default_rng(42), B, m.T, m.dx,
                                  pit.dnc_bridge_count(m.T))
    want = _oracle_paths(oracle, sampler, m, fr_o, term, back, bridge)
    got = lgssm.PathSampler(gm, B, sampler, True)(fr, lgssm.Noise.predrawn(term, back, bridge))
    assert_close(got.cpu(), want, RTOL, f"sampler {sampler}")


def test_kalman_filter_batched_sequences(gpu, oracle):
    lgssm, _, _ = gpu
    m, _ = _oracle_case(oracle, 30, 3, 2, True, True, 11)
    obs = np.stack([simulate_obs(m, oracle.from_seed(500 + i)) for i in range(37)])
    fr = lgssm.kalman_filter(to_gpu_model(m), obs)
    for i in (0, 17, 36):
        want = oracle.kalman_filter(m, obs[i])
        assert_close(fr.filt_mean[i].cpu(), want.filt_mean, RTOL, "filt_mean")
        assert_close(fr.log_marginal[i].cpu(), want.log_marginal, RTOL, "log_marginal")


def _oracle_paths(oracle, sampler, m, fr, term, back, bridge):
    fn = {0: oracle.backward_sample, 1: oracle.prefix_sample, 2: oracle.dnc_sample}[sampler]
    outs = []
    for b in range(term.shape[0]):
        nz, keep = oracle.predrawn_noise(m.dx, term[b], back[b],
                                         None if bridge is None else bridge[b])
        outs.append(fn(m, fr, nz))
    return np.stack(outs)


@pytest.mark.parametrize("sampler", [0, 1, 2])
@pytest.mark.parametrize("case", CASES)
def test_samplers_predrawn_match_oracle(gpu, oracle, sampler, case):
    lgssm, pit, _ = gpu
    m, obs = _oracle_case(oracle, *case)
    fr_o = oracle.kalman_filter(m, obs)
    gm = to_gpu_model(m)
    fr = lgssm.kalman_filter(gm, obs)
    B = 5
    nb = pit.dnc_bridge_count(m.T)
    term, back, bridge = predrawn(np.random.default_rng(case[-1]), B, m.T, m.dx, nb)
    want = _oracle_paths(oracle, sampler, m, fr_o, term, back, bridge)
    noise = lgssm.Noise.predrawn(term, back, bridge)
    got = lgssm.PathSampler(gm, B, sampler, True)(fr, noise)
    assert_close(got.cpu(), want, RTOL, f"sampler {sampler}")


@pytest.mark.parametrize("sampler", [0, 1, 2])
def test_samplers_stream_noise_match_oracle(gpu, oracle, sampler):
    """Device counter RNG vs the oracle's StreamNoise on the same keys."""
    lgssm, _, rng = gpu
    m, obs = _oracle_case(oracle, 77, 4, 1, False, False, 21)
    fr_o = oracle.kalman_filter(m, obs)
    gm = to_gpu_model(m)
    fr = lgssm.kalman_filter(gm, obs)
    keys = rng.chain_keys(200, 6)
    got = lgssm.PathSampler(gm, 6, sampler, True)(fr, lgssm.Noise.stream(keys)).cpu().numpy()
    fn = {0: oracle.backward_sample, 1: oracle.prefix_sample, 2: oracle.dnc_sample}[sampler]
    for c in range(6):
        key = oracle.derive(oracle.from_seed(200), oracle.L_CHAIN, c)
        want = fn(m, fr_o, oracle.stream_noise(key))
        assert_close(got[c], want, RTOL, f"chain {c}")


def test_c2_shape_shared_filter_many_chains(gpu, oracle):
    """One shared filter result, many chains, d = 4 (C2 class at reduced T)."""
    lgssm, _, rng = gpu
    s = oracle.spec("lgssm-synthetic", T=1500, dx=4, dy=1, data_seed=1)
    lat, data = oracle.simulate(s)
    m = oracle.synthetic_lgssm(s)
    fr_o = oracle.kalman_filter(m, data)
    gm = to_gpu_model(m)
    fr = lgssm.kalman_filter(gm, data)
    B = 37
    term, back, _ = predrawn(np.random.default_rng(5), B, m.T, m.dx)
    got = lgssm.PathSampler(gm, B, 1, True)(fr, lgssm.Noise.predrawn(term, back)).cpu().numpy()
    seq = lgssm.PathSampler(gm, B, 0, True)(fr, lgssm.Noise.predrawn(term, back)).cpu().numpy()
    for c in (0, 13, 36):
        nz, keep = oracle.predrawn_noise(4, term[c], back[c])
        want = oracle.prefix_sample(m, fr_o, nz)
        assert_close(got[c], want, RTOL, f"prefix chain {c}")
        assert_close(seq[c], want, 1e-8, f"seq chain {c}")


def test_prefix_is_bit_deterministic(gpu, oracle):
    lgssm, _, rng = gpu
    m, obs = _oracle_case(oracle, 1000, 4, 2, False, False, 31)
    gm = to_gpu_model(m)
    fr = lgssm.kalman_filter(gm, obs)
    keys = rng.chain_keys(9, 20)
    for sampler in (1, 2):
        ps = lgssm.PathSampler(gm, 20, sampler, True)
        a = ps(fr, lgssm.Noise.stream(keys)).clone()
        b = ps(fr, lgssm.Noise.stream(keys))
        assert torch.equal(a, b)


def test_deterministic_dynamics_give_constant_paths(gpu, oracle):
    """Copy dynamics with Q = 0 (test_pit.cpp:242-250, zero-cov fast paths)."""
    lgssm, _, rng = gpu
    T = 12
    m = oracle.Model.homogeneous(T, [0.3], [[1.0]], [[1.0]], [0.0], [[0.0]], [[1.0]], [0.0],
                                 [[0.5]])
    obs = np.linspace(-1, 1, T + 1)[:, None]
    gm = to_gpu_model(m)
    fr = lgssm.kalman_filter(gm, obs)
    for sampler in (0, 1, 2):
        x = lgssm.PathSampler(gm, 3, sampler, True)(fr, lgssm.Noise.stream(rng.chain_keys(1, 3)))
        x = x.cpu().numpy()
        assert np.all(np.abs(x - x[:, -1:, :]) < 1e-10)


def test_per_path_filter_results(gpu, oracle):
    """fr_shared = 0: each path has its own filter result (aux-kernel layout)."""
    lgssm, pit, rng = gpu
    m, _ = _oracle_case(oracle, 60, 3, 1, True, False, 41)
    B = 9
    obs = np.stack([simulate_obs(m, oracle.from_seed(900 + i)) for i in range(B)])
    gm = to_gpu_model(m)
    fr = lgssm.kalman_filter(gm, obs)
    term, back, bridge = predrawn(np.random.default_rng(3), B, m.T, m.dx,
                                  pit.dnc_bridge_count(m.T))
    for sampler in (0, 1, 2):
        got = lgssm.PathSampler(gm, B, sampler, False)(
            fr, lgssm.Noise.predrawn(term, back, bridge)).cpu().numpy()
        for b in (0, 4, 8):
            fr_o = oracle.kalman_filter(m, obs[b])
            want = _oracle_paths(oracle, sampler, m, fr_o, term[b:b + 1], back[b:b + 1],
                                 bridge[b:b + 1])[0]
            assert_close(got[b], want, RTOL, f"sampler {sampler} path {b}")


def test_path_logpdf_matches_oracle(gpu, oracle):
    lgssm, _, rng = gpu
    m, obs = _oracle_case(oracle, 45, 3, 2, True, True, 51)
    fr_o = oracle.kalman_filter(m, obs)
    gm = to_gpu_model(m)
    fr = lgssm.kalman_filter(gm, obs)
    B = 4
    x = lgssm.PathSampler(gm, B, 0, True)(fr, lgssm.Noise.stream(rng.chain_keys(3, B)))
    got = lgssm.path_logpdf(gm, obs, x, fr).cpu().numpy()
    for b in range(B):
        want = oracle.path_logpdf(m, obs, x[b].cpu().numpy(), fr_o)
        assert_close(got[b], want, RTOL, "path_logpdf")


def test_device_normals_match_stream(gpu, oracle):
    _, _, rng = gpu
    keys = rng.chain_keys(4, 3)
    out = rng.normals(keys, 1, 5, 7, 4).cpu().numpy()
    for c in range(3):
        base = oracle.derive(oracle.from_seed(4), oracle.L_CHAIN, c)
        for i in range(7):
            s = oracle.derive(base, 1, 5 + i)
            want = oracle.normal_vec(s, 4)
            assert np.all(np.abs(out[c, i] - want) <= 4e-16 * np.maximum(1, np.abs(want)))


@pytest.mark.parametrize("case", CASES)
def test_parallel_filter_matches_oracle(gpu, oracle, case):
    """pit::parallel_filter (pit.cpp:117-188): GPU blocked scan vs the oracle's
    Sklansky scan and vs the sequential filter (test_pit.cpp:188-229)."""
    lgssm, _, _ = gpu
    m, obs = _oracle_case(oracle, *case)
    seq = oracle.kalman_filter(m, obs)
    par, _ = oracle.parallel_filter(m, obs)
    fr = lgssm.parallel_filter(to_gpu_model(m), obs)
    assert int(fr.status[0]) == 0
    assert_close(fr.filt_mean[0].cpu(), par.filt_mean, 1e-8, "filt_mean vs oracle scan")
    assert_close(fr.filt_cov[0].cpu(), par.filt_cov, 1e-8, "filt_cov vs oracle scan")
    assert_close(fr.pred_cov[0].cpu(), par.pred_cov, 1e-8, "pred_cov vs oracle scan")
    assert_close(fr.log_marginal[0].cpu(), par.log_marginal, 1e-9, "log_marginal")
    assert_close(fr.filt_mean[0].cpu(), seq.filt_mean, 1e-6, "filt_mean vs sequential")


@pytest.mark.parametrize("case", LARGE_CASES[:2] + LARGE_CASES[3:] + [(20, 3, 11, True, True, 36),
                                                                     (40, 9, 4, True, True, 37),
                                                                     (60, 16, 16, True, True, 42),
                                                                     (150, 16, 5, False, True, 43)])
def test_parallel_filter_large_dims_matches_oracle(gpu, oracle, case):
    """Group (warp / CTA) scan filter for dx > 6 or dy > 8: group LU combine,
    element build and recovery vs the oracle's Sklansky scan."""
    lgssm, _, _ = gpu
    m, obs = _oracle_case(oracle, *case)
    par, _ = oracle.parallel_filter(m, obs)
    fr = lgssm.parallel_filter(to_gpu_model(m), obs)
    assert int(fr.status[0]) == 0
    assert_close(fr.filt_mean[0].cpu(), par.filt_mean, 1e-8, "filt_mean vs oracle scan")
    assert_close(fr.filt_cov[0].cpu(), par.filt_cov, 1e-8, "filt_cov vs oracle scan")
    assert_close(fr.pred_mean[0].cpu(), par.pred_mean, 1e-8, "pred_mean vs oracle scan")
    assert_close(fr.pred_cov[0].cpu(), par.pred_cov, 1e-8, "pred_cov vs oracle scan")
    assert_close(fr.log_marginal[0].cpu(), par.log_marginal, 1e-9, "log_marginal")


def test_parallel_filter_generic_two_level_carry(gpu, oracle):
    """Generic scan filter with more than 64 blocks: the block carries are
    themselves scanned in two levels; d = 7 (warp groups), T = 3000."""
    lgssm, _, _ = gpu
    m, obs = _oracle_case(oracle, 3000, 7, 2, False, True, 38)
    seq = oracle.kalman_filter(m, obs)
    fr = lgssm.parallel_filter(to_gpu_model(m), obs)
    assert int(fr.status[0]) == 0
    assert_close(fr.filt_mean[0].cpu(), seq.filt_mean, 1e-8, "filt_mean vs sequential")
    assert_close(fr.filt_cov[0].cpu(), seq.filt_cov, 1e-8, "filt_cov vs sequential")
    assert_close(fr.log_marginal[0].cpu(), seq.log_marginal, 1e-9, "log_marginal")


def test_parallel_filter_batched_long(gpu, oracle):
    lgssm, _, _ = gpu
    s = oracle.spec("lgssm-synthetic", T=5000, dx=4, dy=1, data_seed=1)
    lat, data = oracle.simulate(s)
    m = oracle.synthetic_lgssm(s)
    seq = oracle.kalman_filter(m, data)
    fr = lgssm.parallel_filter(to_gpu_model(m), np.stack([data, data]))
    for b in range(2):
        assert_close(fr.filt_mean[b].cpu(), seq.filt_mean, 1e-8, "filt_mean")
        assert_close(fr.log_marginal[b].cpu(), seq.log_marginal, 1e-9, "log_marginal")


def test_dnc_predrawn_requires_bridge_draws(gpu, oracle):
    """Pre-drawn DnC without the bridge variates is an argument error (AUXMC_E_ARG),
    never a read through a null pointer."""
    lgssm, _, _ = gpu
    m, obs = _oracle_case(oracle, 20, 2, 1, False, False, 3)
    gm = to_gpu_model(m)
    fr = lgssm.kalman_filter(gm, obs)
    term, back, _ = predrawn(np.random.default_rng(0), 2, m.T, m.dx, 32)
    with pytest.raises(Exception):
        lgssm.PathSampler(gm, 2, 2, True)(fr, lgssm.Noise.predrawn(term, back, None))


@pytest.mark.parametrize("sampler", [1, 2])
def test_host_pipeline_equals_device_call(gpu, oracle, sampler):
    """lgssm.HostPipeline (chunked host<->device copies on three streams) returns
    exactly the paths of one device-side PathSampler call."""
    lgssm, pit, _ = gpu
    m, obs = _oracle_case(oracle, 200, 4, 1, False, False, 44)
    gm = to_gpu_model(m)
    fr = lgssm.kalman_filter(gm, obs)
    B = 16
    term, back, bridge = predrawn(np.random.default_rng(9), B, m.T, m.dx,
                                  pit.dnc_bridge_count(m.T))
    noise = lgssm.Noise.predrawn(term, back, bridge if sampler == 2 else None)
    want = lgssm.PathSampler(gm, B, sampler, True)(fr, noise).cpu()
    pin = lambda t: None if t is None else t.cpu().pin_memory()  # noqa: E731
    h_fr = lgssm.FilterResult(pin(fr.pred_mean), pin(fr.pred_cov), pin(fr.filt_mean),
                              pin(fr.filt_cov), pin(fr.log_marginal), fr.status.cpu())
    h_noise = lgssm.Noise(terminal=pin(noise.terminal), backward=pin(noise.backward),
                          bridge=pin(noise.bridge))
    out = torch.empty((B, m.T + 1, m.dx), dtype=torch.float64).pin_memory()
    lgssm.HostPipeline(gm, B, sampler, chunks=4)(h_fr, h_noise, out)
    torch.cuda.synchronize()
    assert torch.equal(out, want)


@pytest.mark.parametrize("T,dx,dy,seed", [(300, 16, 16, 44), (200, 10, 3, 45), (2, 12, 5, 46),
                                          (3000, 10, 3, 47)])
def test_parallel_filter_time_invariant_fill_bit_identical(gpu, oracle, T, dx, dy, seed):
    """Generic scan filter: a model with shared F, b, Q, H, c, R takes the fill
    paths (elements: t = 1 built in full, other steps copy its matrices and form
    their vectors in the same order; block reduction: the matrix sequence run
    once, each block's vectors carried through the combine's formulas); the same
    model given with per-step copies of every matrix takes the full paths.  Results must be identical
    bits, and match the oracle's scan."""
    lgssm, _, _ = gpu
    m, obs = _oracle_case(oracle, T, dx, dy, False, False, seed)
    shared = to_gpu_model(m)
    def rep(a, n):
        return np.repeat(np.asarray(a), n, axis=0)  # shared arrays have a leading 1
    per_step = lgssm.Model(m.T, m.m0, m.P0, rep(m.F, T), rep(m.b, T), rep(m.Q, T),
                           rep(m.H, T + 1), rep(m.c, T + 1), rep(m.R, T + 1), None)
    a = lgssm.parallel_filter(shared, obs)
    b = lgssm.parallel_filter(per_step, obs)
    for name in ("filt_mean", "filt_cov", "pred_mean", "pred_cov", "log_marginal"):
        assert torch.equal(getattr(a, name), getattr(b, name)), name
    ref = oracle.parallel_filter(m, obs)[0] if T < 1000 else oracle.kalman_filter(m, obs)
    assert_close(a.filt_mean[0].cpu(), ref.filt_mean, 1e-8, "filt_mean vs oracle")
    assert_close(a.log_marginal[0].cpu(), ref.log_marginal, 1e-9, "log_marginal")
