"""ctypes binding of the REFERENCE ITSELF (oracle/_ref/libref_bridge.so).

TEST INFRASTRUCTURE ONLY — imported by tests/ and bench.py's CPU legs, never by the
product package.  oracle/_ref/ is the unmodified reference (/root/reference/proj/src)
compiled by oracle/ref.mk against the Eigen / doctest shims in oracle/ref_shim/; this
module exposes its C++ API through the flat C bridge oracle/ref_bridge.cpp with the
same names and argument meanings as oracle/pyoracle.py (the C restatement), so a test
can run one check against both.  `available()` is False where _ref was never built
(the GPU box only has what the container built: the .so files travel with the repo).
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib
import subprocess

import numpy as np

from . import pyoracle as O

HERE = pathlib.Path(__file__).resolve().parent
REF_DIR = HERE / "_ref"
LIB_PATH = REF_DIR / "libref_bridge.so"
REF_SRC = pathlib.Path(os.environ.get("AUXMC_REF_SRC", "/root/reference/proj"))

RB_OK, RB_E_DIM, RB_E_FACTOR, RB_E_DEGENERATE, RB_E_CONTRACT, RB_E_CONFIG = 0, 1, 2, 3, 4, 5
PD, PU8, PU64, PI, PL = O.PD, O.PU8, O.PU64, O.PI, C.POINTER(C.c_long)
VP = C.c_void_p
BACKEND = {"seq": 0, "prefix": 1, "dnc": 2}


def build(jobs: int = 8) -> pathlib.Path:
    """make -f oracle/ref.mk (needs the reference sources; a no-op when up to date)."""
    if not REF_SRC.exists():
        if LIB_PATH.exists():
            return LIB_PATH
        raise RuntimeError(f"reference sources not found at {REF_SRC}")
    r = subprocess.run(["make", "-s", f"-j{jobs}", "-f", str(HERE / "ref.mk"), f"REF={REF_SRC}"],
                       cwd=str(HERE.parent), capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(r.stdout + r.stderr)
    return LIB_PATH


def available() -> bool:
    return LIB_PATH.exists()


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        _lib = C.CDLL(str(LIB_PATH))
        _declare(_lib)
    return _lib


def _declare(L):
    SP = C.POINTER(O.Spec)
    sig = {
        "rb_from_seed": (C.c_uint64, [C.c_uint64]),
        "rb_derive": (C.c_uint64, [C.c_uint64, C.c_uint64, C.c_uint64]),
        "rb_draw": (None, [C.c_uint64, C.c_int, C.c_int, PD, PU64]),
        "rb_simulate": (C.c_int, [SP, PD, PD]),
        "rb_target_new": (VP, [SP, PD, C.c_int, PI]),
        "rb_target_free": (None, [VP]),
        "rb_target_test": (VP, [C.c_int, C.c_int]),
        "rb_target_lgssm": (VP, [VP, PD, C.c_int]),
        "rb_log_gamma": (C.c_double, [VP, PD, PI]),
        "rb_grad_pot": (C.c_int, [VP, C.c_int, PD, C.c_int, PD]),
        "rb_log_pot": (C.c_double, [VP, C.c_int, PD]),
        "rb_lgssm_synthetic": (VP, [SP, PI]),
        "rb_lgssm_new": (VP, [C.c_int, C.c_int, C.c_int, PD, PD, PD, C.c_int, PD, C.c_int, PD,
                              C.c_int, PD, C.c_int, PD, C.c_int, PD, C.c_int, PU8, PI]),
        "rb_lgssm_free": (None, [VP]),
        "rb_filter": (VP, [VP, PD, C.c_int, C.c_int, PI]),
        "rb_filter_get": (None, [VP, PD, PD, PD, PD, PD]),
        "rb_filter_free": (None, [VP]),
        "rb_sample": (C.c_int, [VP, VP, C.c_int, C.c_uint64, PD, PD, PD, C.c_long, C.c_int, PD]),
        "rb_path_logpdf": (C.c_double, [VP, PD, PD, VP, PI]),
        "rb_set_flip_backward_gain": (None, [C.c_int]),
        "rb_aux_chain_new": (VP, [VP, PD, C.c_double, PI]),
        "rb_aux_chain_free": (None, [VP]),
        "rb_aux_step": (C.c_int, [VP, VP, C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int]),
        "rb_aux_adapt": (None, [VP, C.c_double]),
        "rb_aux_get": (None, [VP, PD, PD, PL]),
        "rb_sample_aux_obs": (C.c_int, [PD, C.c_int, C.c_int, C.c_double, C.c_uint64, PD]),
        "rb_mh_log_ratio": (C.c_double, [VP, PD, PD, PD, C.c_double, C.c_int, PI]),
        "rb_pg_new": (VP, [PD, C.c_int, C.c_int, C.c_double]),
        "rb_pg_free": (None, [VP]),
        "rb_pg_step": (C.c_int, [VP, VP, C.c_int, C.c_uint64, C.c_int, PI]),
        "rb_pg_adapt": (None, [VP, C.c_double]),
        "rb_pg_step_pm": (C.c_int, [VP, VP, C.c_int, C.c_uint64, C.c_int, C.c_int, PI]),
        "rb_pg_get": (None, [VP, PD, PU64, PD, PL]),
        "rb_csmc_trace": (C.c_int, [VP, PD, PU64, PD, C.c_double, C.c_int, C.c_uint64, C.c_int,
                                    PI, PD, PI]),
        "rb_run_json": (C.c_int, [C.c_char_p, PD]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


_p, _f64 = O._p, O._f64


def _check(st, what):
    if st != RB_OK:
        raise RuntimeError(f"{what}: reference status {st}")


def _key(s) -> int:
    return int(s.key) if hasattr(s, "key") else int(s)


# ---------------------------------------------------------------- RNG (rng.hpp)
def from_seed_key(seed: int) -> int:
    return lib().rb_from_seed(seed)


def derive_key(key: int, label: int, index: int) -> int:
    return lib().rb_derive(_key(key), label, index)


def draws(key, kind: str, n: int):
    """First n draws of the stream with this key: 'normal', 'uniform' or 'key'."""
    k = {"normal": 0, "uniform": 1, "key": 2}[kind]
    out, out_u = np.zeros(n), np.zeros(n, np.uint64)
    lib().rb_draw(_key(key), k, n, _p(out), out_u.ctypes.data_as(PU64))
    return out_u if k == 2 else out


# ---------------------------------------------------------------- models (models.cpp)
def simulate(s: O.Spec):
    dx, dy = O.latent_dim(s), O.obs_dim(s)
    lat = np.zeros((s.T + 1, dx))
    data = np.zeros((s.T + 1, max(dy, 0)))
    _check(lib().rb_simulate(C.byref(s), _p(lat), _p(data) if data.size else _p(np.zeros(1))),
           "simulate")
    return lat, data


class RTarget:
    """Reference GenSSMTarget built by bench::make_target (models.cpp:240-336), or the
    Lorenz-96 target on GenSSMTarget::tractable (kind "lorenz96")."""

    def __init__(self, s: O.Spec, data):
        self.data = _f64(data)
        self.T, self.dx = s.T, O.latent_dim(s)
        ydim = self.data.shape[1] if self.data.ndim == 2 else 0
        st = C.c_int(0)
        self.h = lib().rb_target_new(C.byref(s), _p(self.data) if self.data.size else
                                     _p(np.zeros(1)), ydim, C.byref(st))
        _check(st.value, "make_target")

    def __del__(self):
        try:
            lib().rb_target_free(self.h)
        except Exception:
            pass

    def log_gamma(self, traj):
        st = C.c_int(0)
        v = lib().rb_log_gamma(self.h, _p(_f64(traj)), C.byref(st))
        _check(st.value, "log_gamma")
        return v

    def grad_pot_generic(self, t, x):
        out = np.zeros(self.dx)
        _check(lib().rb_grad_pot(self.h, t, _p(_f64(x)), 1, _p(out)), "grad_pot_generic")
        return out

    def grad_pot(self, t, x):
        out = np.zeros(self.dx)
        _check(lib().rb_grad_pot(self.h, t, _p(_f64(x)), 0, _p(out)), "grad_pot")
        return out

    def log_pot(self, t, x):
        return lib().rb_log_pot(self.h, t, _p(_f64(x)))


def make_target(s: O.Spec, data) -> RTarget:
    return RTarget(s, data)


def target_from_lgssm(m, obs, generic=False) -> RTarget:
    """testutil.hpp:88-140: the LGSSM posterior with exact or generic potentials."""
    rm = model(m)
    t = RTarget.__new__(RTarget)
    t.T, t.dx, t.data = rm.T, rm.dx, _f64(obs)
    t._model = rm
    t.h = lib().rb_target_lgssm(rm.h, _p(t.data), int(generic))
    return t


def test_target(name: str, T: int) -> RTarget:
    """The reference's failure-path test targets (ref_bridge.cpp rb_target_test)."""
    t = RTarget.__new__(RTarget)
    t.T, t.dx, t.data = T, 1, np.zeros(0)
    t.h = lib().rb_target_test({"test-abort": 7, "test-support": 8, "test-collapse": 9}[name], T)
    return t


class RModel:
    """Reference lgssm::Model (lgssm.cpp:20-71) from a pyoracle.Model's arrays."""

    def __init__(self, m: O.Model):
        self.src = m
        self.T, self.dx, self.dy = m.T, m.dx, m.dy
        st = C.c_int(0)
        self.h = lib().rb_lgssm_new(
            m.T, m.dx, m.dy, _p(m.m0), _p(m.P0), _p(m.F), m.F.shape[0], _p(m.b), m.b.shape[0],
            _p(m.Q), m.Q.shape[0], _p(m.H), m.H.shape[0], _p(m.c), m.c.shape[0], _p(m.R),
            m.R.shape[0], m.mask.ctypes.data_as(PU8) if m.mask is not None else None,
            C.byref(st))
        _check(st.value, "Model")

    def __del__(self):
        try:
            lib().rb_lgssm_free(self.h)
        except Exception:
            pass


def model(m) -> RModel:
    return m if isinstance(m, RModel) else RModel(m)


class RFilter:
    def __init__(self, h, T, dx):
        self.h = h
        self.pred_mean, self.filt_mean = np.zeros((T + 1, dx)), np.zeros((T + 1, dx))
        self.pred_cov, self.filt_cov = np.zeros((T + 1, dx, dx)), np.zeros((T + 1, dx, dx))
        lm = np.zeros(1)
        lib().rb_filter_get(h, _p(self.pred_mean), _p(self.pred_cov), _p(self.filt_mean),
                            _p(self.filt_cov), _p(lm))
        self.log_marginal = float(lm[0])

    def __del__(self):
        try:
            lib().rb_filter_free(self.h)
        except Exception:
            pass


def _filter(m, obs, parallel, workers=1) -> RFilter:
    rm = model(m)
    st = C.c_int(0)
    h = lib().rb_filter(rm.h, _p(_f64(obs)), int(parallel), workers, C.byref(st))
    _check(st.value, "filter")
    return RFilter(h, rm.T, rm.dx)


def kalman_filter(m, obs) -> RFilter:
    """lgssm.cpp:73-112"""
    return _filter(m, obs, False)


def parallel_filter(m, obs, workers=1) -> RFilter:
    """pit.cpp:117-188"""
    return _filter(m, obs, True, workers)


def _sample(which, m, fr: RFilter, noise, workers=1):
    rm = model(m)
    out = np.zeros((rm.T + 1, rm.dx))
    if isinstance(noise, dict):  # pre-drawn: terminal [dx], backward [T][dx], bridge [n][dx]
        term, bwd = _f64(noise["terminal"]), _f64(noise["backward"])
        br = noise.get("bridge")
        br = _f64(br) if br is not None else None
        st = lib().rb_sample(rm.h, fr.h, which, 0, _p(term), _p(bwd), _p(br),
                             br.shape[0] if br is not None else 0, workers, _p(out))
    else:  # StreamNoise over this stream (rng.hpp:128-137)
        st = lib().rb_sample(rm.h, fr.h, which, _key(noise), None, None, None, 0, workers,
                             _p(out))
    _check(st, "sample")
    return out


def backward_sample(m, fr, noise):
    return _sample(0, m, fr, noise)


def prefix_sample(m, fr, noise, workers=1):
    return _sample(1, m, fr, noise, workers)


def dnc_sample(m, fr, noise, workers=1):
    return _sample(2, m, fr, noise, workers)


def path_logpdf(m, obs, traj, fr: RFilter) -> float:
    rm = model(m)
    st = C.c_int(0)
    v = lib().rb_path_logpdf(rm.h, _p(_f64(obs)), _p(_f64(traj)), fr.h, C.byref(st))
    _check(st.value, "path_logpdf")
    return v


def set_flip_backward_gain(on: bool):
    lib().rb_set_flip_backward_gain(int(on))


# ---------------------------------------------------------------- aux Kalman (auxk.cpp)
class AuxChain:
    """AuxChainState + kernel_step (auxk.cpp:120-198); step(root) takes the chain root
    stream (the iteration stream is root.derive(kIteration, iter), auxk.cpp:131)."""

    def __init__(self, tg: RTarget, x0, delta):
        self.tg = tg
        st = C.c_int(0)
        self.h = lib().rb_aux_chain_new(tg.h, _p(_f64(x0)), delta, C.byref(st))
        _check(st.value, "init_chain")

    def __del__(self):
        try:
            lib().rb_aux_chain_free(self.h)
        except Exception:
            pass

    def step(self, root, backend=0, parallel_filter=0, zeroth_order=0, workers=1):
        _check(lib().rb_aux_step(self.tg.h, self.h, _key(root), backend, int(parallel_filter),
                                 int(zeroth_order), workers), "kernel_step")

    def adapt(self, target_rate):
        lib().rb_aux_adapt(self.h, target_rate)

    def state(self, with_x=True):
        x = np.zeros((self.tg.T + 1, self.tg.dx)) if with_x else None
        sc, ints = np.zeros(4), np.zeros(5, np.int64)
        lib().rb_aux_get(self.h, _p(x), _p(sc), ints.ctypes.data_as(PL))
        return dict(x=x, delta=sc[0], log_gamma=sc[1], last_log_alpha=sc[2],
                    last_accept_prob=sc[3], accepted=int(ints[0]), rejected=int(ints[1]),
                    aborted=int(ints[2]), nonfinite_gamma=int(ints[3]), iter=int(ints[4]))

    @property
    def x(self):
        return self.state()["x"]


def sample_aux_obs(x, delta, it):
    x = _f64(x)
    u = np.zeros_like(x)
    _check(lib().rb_sample_aux_obs(_p(x), x.shape[0] - 1, x.shape[1], delta, _key(it), _p(u)),
           "sample_aux_obs")
    return u


def mh_log_ratio(tg: RTarget, x, xp, u, delta, zeroth_order=False):
    st = C.c_int(0)
    v = lib().rb_mh_log_ratio(tg.h, _p(_f64(x)), _p(_f64(xp)), _p(_f64(u)), delta,
                              int(zeroth_order), C.byref(st))
    _check(st.value, "mh_log_ratio")
    return v


# ---------------------------------------------------------------- particle Gibbs (fkpg.cpp)
class PGChain:
    def __init__(self, tg: RTarget, x0, delta):
        self.tg = tg
        self.h = lib().rb_pg_new(_p(_f64(x0)), tg.T, tg.dx, delta)

    def __del__(self):
        try:
            lib().rb_pg_free(self.h)
        except Exception:
            pass

    def step(self, N, root, mode=1, pm=0):
        """aux_pgibbs_step; returns (status, bad_t).  pm: the pseudo-marginal estimator
        (fkpg.cpp:233-250) of the reference's tests, see rb_pg_step_pm."""
        bad = C.c_int(-1)
        if pm:
            st = lib().rb_pg_step_pm(self.tg.h, self.h, N, _key(root), mode, pm, C.byref(bad))
        else:
            st = lib().rb_pg_step(self.tg.h, self.h, N, _key(root), mode, C.byref(bad))
        return st, bad.value

    def adapt(self, target_rate):
        lib().rb_pg_adapt(self.h, target_rate)

    def state(self):
        x = np.zeros((self.tg.T + 1, self.tg.dx))
        keys = np.zeros(self.tg.T + 1, np.uint64)
        sc, ints = np.zeros(2), np.zeros(2, np.int64)
        lib().rb_pg_get(self.h, _p(x), keys.ctypes.data_as(PU64), _p(sc), ints.ctypes.data_as(PL))
        return dict(x=x, keys=keys, delta=sc[0], last_update=sc[1], iter=int(ints[0]),
                    updates=int(ints[1]))

    @property
    def x(self):
        return self.state()["x"]

    @property
    def keys(self):
        return self.state()["keys"]


def csmc_trace(tg: RTarget, ref, ref_keys, u, delta, N, it, mode=1):
    """csmc_step over build_aux_fk: (status, bad_t, ancestors [T+1][N], traj)."""
    T = tg.T
    anc = np.zeros((T + 1, N), np.int32)
    traj = np.zeros((T + 1, tg.dx))
    rk = np.ascontiguousarray(np.asarray(ref_keys, np.uint64))
    bad = C.c_int(-1)
    st = lib().rb_csmc_trace(tg.h, _p(_f64(ref)), rk.ctypes.data_as(PU64), _p(_f64(u)), delta, N,
                             _key(it), mode, anc.ctypes.data_as(PI), _p(traj), C.byref(bad))
    return st, bad.value, anc, traj


def run_json(text: str) -> float:
    """bench::run (runner.cpp:112-244) on a JSON run config; returns the summary rate."""
    rate = np.zeros(1)
    _check(lib().rb_run_json(text.encode(), _p(rate)), "run")
    return float(rate[0])
