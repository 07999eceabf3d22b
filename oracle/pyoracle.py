"""ctypes binding of the CPU parity oracle (oracle/build/liboracle.so).

TEST INFRASTRUCTURE ONLY — imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py, never by the product package.
Arrays are numpy float64, row-major, shapes as in auxmc_oracle.h.
"""
from __future__ import annotations

import ctypes as C
import pathlib
import subprocess

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = HERE / "build" / "liboracle.so"

AO_OK, AO_E_DIM, AO_E_FACTOR, AO_E_DEGENERATE = 0, 1, 2, 3
KIND = {"lgssm-synthetic": 0, "stochvol": 1, "diffusion-smoothing": 2, "spatio-temporal": 3,
        "grid-1d-test": 4, "lorenz96": 5, "gauss-generic": 6}
L_BACKWARD_NOISE, L_TERMINAL_DRAW, L_AUX_OBS, L_DNC_BRIDGE, L_MH_ACCEPT = 1, 2, 3, 4, 5
L_ITERATION, L_CHAIN, L_STEP, L_PARTICLE, L_RESAMPLE = 6, 7, 8, 9, 10
L_TERMINAL_INDEX, L_BACKWARD_INDEX, L_PM_KEY, L_SIMULATE, L_PARAM = 11, 12, 13, 14, 15


def build():
    r = subprocess.run(["make", "-s", "-C", str(HERE)], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(r.stdout + r.stderr)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        _lib = C.CDLL(str(LIB_PATH))
        _declare(_lib)
    return _lib


PD = C.POINTER(C.c_double)
PU8 = C.POINTER(C.c_uint8)
PU64 = C.POINTER(C.c_uint64)
PI = C.POINTER(C.c_int)


class Stream(C.Structure):
    _fields_ = [("key", C.c_uint64), ("counter", C.c_uint64)]


class Noise(C.Structure):
    _fields_ = [("kind", C.c_int), ("base", Stream), ("dx", C.c_int), ("terminal", PD),
                ("backward", PD), ("n_backward", C.c_long), ("bridge", PD),
                ("n_bridge", C.c_long), ("active", C.c_int), ("cursor", C.c_int)]


class LGSSM(C.Structure):
    _fields_ = [("T", C.c_int), ("dx", C.c_int), ("dy", C.c_int), ("m0", PD), ("P0", PD),
                ("F", PD), ("b", PD), ("Q", PD), ("H", PD), ("c", PD), ("R", PD),
                ("nF", C.c_int), ("nb", C.c_int), ("nQ", C.c_int), ("nH", C.c_int),
                ("nc", C.c_int), ("nR", C.c_int), ("mask", PU8)]


class Filter(C.Structure):
    _fields_ = [("pred_mean", PD), ("pred_cov", PD), ("filt_mean", PD), ("filt_cov", PD),
                ("log_marginal", C.c_double)]


class Spec(C.Structure):
    _fields_ = [("kind", C.c_int), ("T", C.c_int), ("dx", C.c_int), ("dy", C.c_int),
                ("grid", C.c_int), ("data_seed", C.c_uint64)] + [
        (n, C.c_double) for n in (
            "sv_mu sv_phi sv_sig2 sv_rho lz_sigma lz_rho lz_beta lz_h lz_gamma lz_obs_var "
            "st_phi st_kappa2 st_tau2 g1_phi g1_q g1_m0 g1_p0 l96_F l96_h l96_gamma "
            "l96_obs_var").split()]


class Target(C.Structure):
    _fields_ = [("kind", C.c_int), ("T", C.c_int), ("dx", C.c_int), ("ydim", C.c_int),
                ("linear", C.c_int), ("m0", PD), ("P0", PD), ("F", PD), ("b", PD), ("Q", PD),
                ("nF", C.c_int), ("q", C.c_int), ("ne", C.c_int), ("eH", PD), ("ec", PD),
                ("eR", PD), ("ey", PD), ("emask", PU8), ("data", PD), ("gmask", PU8),
                ("spec", Spec)]


class KStats(C.Structure):
    _fields_ = [("accepted", C.c_long), ("rejected", C.c_long), ("aborted", C.c_long),
                ("nonfinite_gamma", C.c_long), ("last_log_alpha", C.c_double),
                ("last_accept_prob", C.c_double)]


class Chain(C.Structure):
    _fields_ = [("x", PD), ("delta", C.c_double), ("log_gamma", C.c_double), ("grad_gen", PD),
                ("iter", C.c_long), ("stats", KStats)]


class PG(C.Structure):
    _fields_ = [("x", PD), ("keys", PU64), ("delta", C.c_double), ("iter", C.c_long),
                ("updates", C.c_long), ("last_update", C.c_double)]


def _declare(L):
    L.ao_mix64.restype = C.c_uint64
    L.ao_mix64.argtypes = [C.c_uint64]
    L.ao_from_seed.restype = Stream
    L.ao_from_seed.argtypes = [C.c_uint64]
    L.ao_derive.restype = Stream
    L.ao_derive.argtypes = [Stream, C.c_uint64, C.c_uint64]
    L.ao_next_uniform.restype = C.c_double
    L.ao_next_uniform.argtypes = [C.POINTER(Stream)]
    L.ao_next_normal.restype = C.c_double
    L.ao_next_normal.argtypes = [C.POINTER(Stream)]
    L.ao_next_key.restype = C.c_uint64
    L.ao_next_key.argtypes = [C.POINTER(Stream)]
    L.ao_normal_vec.argtypes = [C.POINTER(Stream), C.c_int, PD]
    L.ao_log_pdf.restype = C.c_double
    L.ao_log_pdf.argtypes = [C.c_int, PD, PD, PD, PI]
    L.ao_isotropic_log_pdf.restype = C.c_double
    L.ao_isotropic_log_pdf.argtypes = [C.c_int, PD, C.c_double]
    L.ao_chol_psd.argtypes = [C.c_int, PD, PD]
    L.ao_solve_spd.argtypes = [C.c_int, PD, C.c_int, PD, PD]
    L.ao_spectral_radius.restype = C.c_double
    L.ao_spectral_radius.argtypes = [C.c_int, PD]
    L.ao_kalman_filter.argtypes = [C.POINTER(LGSSM), PD, C.POINTER(Filter)]
    L.ao_parallel_filter.argtypes = [C.POINTER(LGSSM), PD, C.POINTER(Filter), PI,
                                     C.POINTER(C.c_long)]
    L.ao_backward_sample.argtypes = [C.POINTER(LGSSM), C.POINTER(Filter), C.POINTER(Noise), PD]
    L.ao_prefix_sample.argtypes = [C.POINTER(LGSSM), C.POINTER(Filter), C.POINTER(Noise), PD,
                                   PI, C.POINTER(C.c_long)]
    L.ao_dnc_sample.argtypes = [C.POINTER(LGSSM), C.POINTER(Filter), C.POINTER(Noise), PD]
    L.ao_rts_smoother.argtypes = [C.POINTER(LGSSM), C.POINTER(Filter), PD, PD]
    L.ao_path_logpdf.restype = C.c_double
    L.ao_path_logpdf.argtypes = [C.POINTER(LGSSM), PD, PD, C.POINTER(Filter), PI]
    L.ao_dense_oracle.argtypes = [C.POINTER(LGSSM), PD, C.c_int, PD, PD, PD]
    L.ao_extract_affine_law.argtypes = [C.c_int, C.POINTER(LGSSM), C.POINTER(Filter), PD, PD]
    L.ao_backward_step.argtypes = [C.POINTER(LGSSM), C.POINTER(Filter), C.c_int, PD, PD, PD]
    L.ao_spec_default.argtypes = [C.POINTER(Spec)]
    L.ao_latent_dim.argtypes = [C.POINTER(Spec)]
    L.ao_obs_dim.argtypes = [C.POINTER(Spec)]
    L.ao_simulate.argtypes = [C.POINTER(Spec), PD, PD]
    L.ao_synth_mats.argtypes = [C.POINTER(Spec), PD, PD, PD, PD, PD, PD, PD]
    L.ao_make_target.argtypes = [C.POINTER(Spec), PD, C.POINTER(Target)]
    L.ao_target_from_lgssm.argtypes = [C.POINTER(LGSSM), PD, C.c_int, C.POINTER(Target)]
    L.ao_target_free.argtypes = [C.POINTER(Target)]
    L.ao_log_gamma.restype = C.c_double
    L.ao_log_gamma.argtypes = [C.POINTER(Target), PD, PI]
    L.ao_grad_pot_generic.argtypes = [C.POINTER(Target), C.c_int, PD, PD]
    L.ao_grad_pot.argtypes = [C.POINTER(Target), C.c_int, PD, PD, PI]
    L.ao_log_pot.restype = C.c_double
    L.ao_log_pot.argtypes = [C.POINTER(Target), C.c_int, PD, PI]
    L.ao_init_chain.argtypes = [C.POINTER(Target), PD, C.c_double, C.POINTER(Chain)]
    L.ao_chain_free.argtypes = [C.POINTER(Chain)]
    L.ao_kernel_step.argtypes = [C.POINTER(Target), C.POINTER(Chain), Stream, C.c_int, C.c_int,
                                 C.c_int]
    L.ao_adapt_delta.argtypes = [C.POINTER(Chain), C.c_double]
    L.ao_gamma_move.argtypes = [C.POINTER(Target), PD, C.POINTER(C.c_double), C.c_double, Stream]
    L.ao_mh_log_ratio.restype = C.c_double
    L.ao_mh_log_ratio.argtypes = [C.POINTER(Target), PD, PD, PD, C.c_double, C.c_int, PI]
    L.ao_sample_aux_obs.argtypes = [PD, C.c_int, C.c_int, C.c_double, Stream, PD]
    L.ao_init_pg.argtypes = [C.POINTER(Target), PD, C.c_double, C.POINTER(PG)]
    L.ao_pg_free.argtypes = [C.POINTER(PG)]
    L.ao_aux_pgibbs_step.argtypes = [C.POINTER(Target), C.POINTER(PG), C.c_int, Stream, C.c_int,
                                     PI, PI, PI]
    L.ao_pg_adapt_delta.argtypes = [C.POINTER(PG), C.c_double]
    L.ao_pit_pgibbs_step.argtypes = [C.POINTER(Target), C.POINTER(PG), C.c_int, Stream, PI, PI]
    L.ao_pit_csmc_marginals.argtypes = [C.POINTER(Target), PD, C.c_double, PD, C.c_int, PD]


def _p(a):
    return a.ctypes.data_as(PD) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


# ---------------------------------------------------------------- RNG
def from_seed(seed: int) -> Stream:
    return lib().ao_from_seed(seed)


def derive(s: Stream, label: int, index: int) -> Stream:
    return lib().ao_derive(s, label, index)


def mix64(z: int) -> int:
    return lib().ao_mix64(z)


def normal_vec(s: Stream, d: int) -> np.ndarray:
    out = np.empty(d)
    lib().ao_normal_vec(C.byref(s), d, _p(out))
    return out


def next_uniform(s: Stream) -> float:
    return lib().ao_next_uniform(C.byref(s))


def next_normal(s: Stream) -> float:
    return lib().ao_next_normal(C.byref(s))


# ---------------------------------------------------------------- LGSSM
class Model:
    """Owned numpy copy of an LGSSM in the oracle's layout (lgssm.hpp:19-49)."""

    def __init__(self, T, m0, P0, F, b, Q, H, c, R, mask=None):
        self.T = int(T)
        self.m0 = _f64(m0)
        self.dx = self.m0.shape[0]
        self.P0 = _f64(P0).reshape(self.dx, self.dx)
        self.F = _f64(F).reshape(-1, self.dx, self.dx)
        self.b = _f64(b).reshape(-1, self.dx)
        self.Q = _f64(Q).reshape(-1, self.dx, self.dx)
        H = _f64(H)
        self.dy = H.shape[-2] if H.size else 0
        self.H = H.reshape(-1, self.dy, self.dx)
        self.c = _f64(c).reshape(-1, self.dy)
        self.R = _f64(R).reshape(-1, self.dy, self.dy)
        self.mask = None if mask is None else np.ascontiguousarray(np.asarray(mask, np.uint8))

    @staticmethod
    def homogeneous(T, m0, P0, F, b, Q, H, c, R, mask=None):
        return Model(T, m0, P0, [F], [b], [Q], [H], [c], [R], mask)

    def raw(self) -> LGSSM:
        m = LGSSM()
        m.T, m.dx, m.dy = self.T, self.dx, self.dy
        m.m0, m.P0 = _p(self.m0), _p(self.P0)
        m.F, m.b, m.Q = _p(self.F), _p(self.b), _p(self.Q)
        m.H, m.c, m.R = _p(self.H), _p(self.c), _p(self.R)
        m.nF, m.nb, m.nQ = self.F.shape[0], self.b.shape[0], self.Q.shape[0]
        m.nH, m.nc, m.nR = self.H.shape[0], self.c.shape[0], self.R.shape[0]
        m.mask = self.mask.ctypes.data_as(PU8) if self.mask is not None else None
        return m

    def observed(self, t):
        return self.mask is None or self.mask[t] != 0


class FilterResult:
    def __init__(self, T, dx):
        self.pred_mean = np.zeros((T + 1, dx))
        self.pred_cov = np.zeros((T + 1, dx, dx))
        self.filt_mean = np.zeros((T + 1, dx))
        self.filt_cov = np.zeros((T + 1, dx, dx))
        self.log_marginal = 0.0

    def raw(self) -> Filter:
        f = Filter()
        f.pred_mean, f.pred_cov = _p(self.pred_mean), _p(self.pred_cov)
        f.filt_mean, f.filt_cov = _p(self.filt_mean), _p(self.filt_cov)
        f.log_marginal = self.log_marginal
        return f


def _check(st, what):
    if st != AO_OK:
        raise RuntimeError(f"{what}: oracle status {st}")


def kalman_filter(m: Model, obs) -> FilterResult:
    obs = _f64(obs)
    fr = FilterResult(m.T, m.dx)
    raw = fr.raw()
    mr = m.raw()
    _check(lib().ao_kalman_filter(C.byref(mr), _p(obs), C.byref(raw)), "kalman_filter")
    fr.log_marginal = raw.log_marginal
    return fr


def parallel_filter(m: Model, obs):
    obs = _f64(obs)
    fr = FilterResult(m.T, m.dx)
    raw = fr.raw()
    mr = m.raw()
    cp = C.c_int(0)
    ap = C.c_long(0)
    _check(lib().ao_parallel_filter(C.byref(mr), _p(obs), C.byref(raw), C.byref(cp), C.byref(ap)),
           "parallel_filter")
    fr.log_marginal = raw.log_marginal
    return fr, (cp.value, ap.value)


def stream_noise(key_stream: Stream) -> Noise:
    n = Noise()
    n.kind = 0
    n.base = key_stream
    return n


def predrawn_noise(dx, terminal, backward, bridge=None) -> tuple:
    n = Noise()
    n.kind = 1
    n.dx = dx
    terminal = _f64(terminal)
    backward = _f64(backward)
    n.terminal = _p(terminal)
    n.backward = _p(backward)
    n.n_backward = backward.shape[0] if backward.ndim > 1 else 0
    keep = [terminal, backward]
    if bridge is not None:
        bridge = _f64(bridge)
        keep.append(bridge)
        n.bridge = _p(bridge)
        n.n_bridge = bridge.shape[0]
    return n, keep


def _sample(fn, m: Model, fr: FilterResult, noise: Noise, *extra):
    out = np.zeros((m.T + 1, m.dx))
    mr, fr_raw = m.raw(), fr.raw()
    st = fn(C.byref(mr), C.byref(fr_raw), C.byref(noise), _p(out), *extra)
    _check(st, fn.__name__)
    return out


def backward_sample(m, fr, noise):
    return _sample(lib().ao_backward_sample, m, fr, noise)


def prefix_sample(m, fr, noise, stats=False):
    cp = C.c_int(0)
    ap = C.c_long(0)
    out = _sample(lib().ao_prefix_sample, m, fr, noise, C.byref(cp), C.byref(ap))
    return (out, (cp.value, ap.value)) if stats else out


def dnc_sample(m, fr, noise):
    return _sample(lib().ao_dnc_sample, m, fr, noise)


def path_logpdf(m, obs, traj, fr) -> float:
    obs, traj = _f64(obs), _f64(traj)
    st = C.c_int(0)
    mr, fr_raw = m.raw(), fr.raw()
    v = lib().ao_path_logpdf(C.byref(mr), _p(obs), _p(traj), C.byref(fr_raw), C.byref(st))
    _check(st.value, "path_logpdf")
    return v


def dense_oracle(m, obs, cap=256):
    obs = _f64(obs)
    n = (m.T + 1) * m.dx
    mean, cov, le = np.zeros(n), np.zeros((n, n)), np.zeros(1)
    mr = m.raw()
    _check(lib().ao_dense_oracle(C.byref(mr), _p(obs), cap, _p(mean), _p(cov), _p(le)),
           "dense_oracle")
    return mean, cov, float(le[0])


def extract_affine_law(which: int, m, fr):
    n = (m.T + 1) * m.dx
    mean, cov = np.zeros(n), np.zeros((n, n))
    mr, fr_raw = m.raw(), fr.raw()
    _check(lib().ao_extract_affine_law(which, C.byref(mr), C.byref(fr_raw), _p(mean), _p(cov)),
           "extract_affine_law")
    return mean, cov


def rts_smoother(m, fr):
    mean, cov = np.zeros((m.T + 1, m.dx)), np.zeros((m.T + 1, m.dx, m.dx))
    mr, fr_raw = m.raw(), fr.raw()
    _check(lib().ao_rts_smoother(C.byref(mr), C.byref(fr_raw), _p(mean), _p(cov)), "rts")
    return mean, cov


def backward_step(m, fr, t):
    G, off, cov = np.zeros((m.dx, m.dx)), np.zeros(m.dx), np.zeros((m.dx, m.dx))
    mr, fr_raw = m.raw(), fr.raw()
    _check(lib().ao_backward_step(C.byref(mr), C.byref(fr_raw), t, _p(G), _p(off), _p(cov)), "bs")
    return G, off, cov


def log_pdf(x, mean, cov):
    x, mean, cov = _f64(x), _f64(mean), _f64(cov)
    st = C.c_int(0)
    v = lib().ao_log_pdf(x.shape[0], _p(x), _p(mean), _p(cov), C.byref(st))
    _check(st.value, "log_pdf")
    return v


def chol_psd(a):
    a = _f64(a)
    out = np.zeros_like(a)
    _check(lib().ao_chol_psd(a.shape[0], _p(a), _p(out)), "chol_psd")
    return out


def spectral_radius(a):
    a = _f64(a)
    return lib().ao_spectral_radius(a.shape[0], _p(a))


# ---------------------------------------------------------------- models / targets
def spec(kind="lgssm-synthetic", **kw) -> Spec:
    s = Spec()
    lib().ao_spec_default(C.byref(s))
    s.kind = KIND[kind] if isinstance(kind, str) else kind
    for k, v in kw.items():
        setattr(s, k, v)
    return s


def latent_dim(s):
    return lib().ao_latent_dim(C.byref(s))


def obs_dim(s):
    return lib().ao_obs_dim(C.byref(s))


def simulate(s: Spec):
    dx, dy = latent_dim(s), obs_dim(s)
    lat = np.zeros((s.T + 1, dx))
    data = np.zeros((s.T + 1, max(dy, 0)))
    _check(lib().ao_simulate(C.byref(s), _p(lat), _p(data) if data.size else _p(np.zeros(1))),
           "simulate")
    return lat, data


def synth_mats(s: Spec):
    dx, dy = s.dx, s.dy
    m0, b, P0, F, Q = np.zeros(dx), np.zeros(dx), np.zeros((dx, dx)), np.zeros((dx, dx)), np.zeros((dx, dx))
    H, R = np.zeros((dy, dx)), np.zeros((dy, dy))
    _check(lib().ao_synth_mats(C.byref(s), _p(m0), _p(b), _p(P0), _p(F), _p(Q), _p(H), _p(R)),
           "synth_mats")
    return dict(m0=m0, b=b, P0=P0, F=F, Q=Q, H=H, R=R)


def synthetic_lgssm(s: Spec) -> Model:
    """models.cpp:338-344"""
    mm = synth_mats(s)
    return Model.homogeneous(s.T, mm["m0"], mm["P0"], mm["F"], mm["b"], mm["Q"], mm["H"],
                             np.zeros(s.dy), mm["R"])


class OTarget:
    """Owned oracle target (target.hpp:34-93)."""

    def __init__(self, raw: Target, keep=()):
        self.raw = raw
        self._keep = keep
        self.T, self.dx = raw.T, raw.dx

    def __del__(self):
        try:
            lib().ao_target_free(C.byref(self.raw))
        except Exception:
            pass

    def log_gamma(self, traj):
        traj = _f64(traj)
        st = C.c_int(0)
        v = lib().ao_log_gamma(C.byref(self.raw), _p(traj), C.byref(st))
        _check(st.value, "log_gamma")
        return v

    def grad_pot_generic(self, t, x):
        x = _f64(x)
        g = np.zeros(self.dx)
        lib().ao_grad_pot_generic(C.byref(self.raw), t, _p(x), _p(g))
        return g

    def grad_pot(self, t, x):
        x = _f64(x)
        g = np.zeros(self.dx)
        st = C.c_int(0)
        lib().ao_grad_pot(C.byref(self.raw), t, _p(x), _p(g), C.byref(st))
        return g

    def log_pot(self, t, x):
        x = _f64(x)
        st = C.c_int(0)
        return lib().ao_log_pot(C.byref(self.raw), t, _p(x), C.byref(st))

    def arrays(self):
        """Flat copies of the target's arrays (for handing to the GPU product)."""
        r = self.raw
        T, dx, q, ne, yd, nF = r.T, r.dx, r.q, r.ne, r.ydim, r.nF
        rows = yd if r.kind == KIND["gauss-generic"] else q

        def arr(ptr, n):
            return np.ctypeslib.as_array(ptr, shape=(n,)).copy() if (ptr and n > 0) else np.zeros(0)
        out = dict(kind=r.kind, T=T, dx=dx, ydim=yd, linear=r.linear, q=q, ne=ne, nF=nF,
                   m0=arr(r.m0, dx), P0=arr(r.P0, dx * dx), F=arr(r.F, nF * dx * dx),
                   b=arr(r.b, nF * dx), Q=arr(r.Q, nF * dx * dx),
                   eH=arr(r.eH, ne * rows * dx), ec=arr(r.ec, ne * rows),
                   eR=arr(r.eR, ne * rows * rows), ey=arr(r.ey, (T + 1) * q),
                   data=arr(r.data, (T + 1) * yd),
                   emask=np.ctypeslib.as_array(r.emask, shape=(T + 1,)).copy(),
                   gmask=np.ctypeslib.as_array(r.gmask, shape=(T + 1,)).copy(),
                   spec=r.spec)
        return out


def make_target(s: Spec, data) -> OTarget:
    data = _f64(data)
    t = Target()
    _check(lib().ao_make_target(C.byref(s), _p(data) if data.size else _p(np.zeros(1)),
                                C.byref(t)), "make_target")
    return OTarget(t)


def target_from_lgssm(m: Model, obs, generic=False) -> OTarget:
    obs = _f64(obs)
    t = Target()
    mr = m.raw()
    _check(lib().ao_target_from_lgssm(C.byref(mr), _p(obs), int(generic), C.byref(t)), "target")
    return OTarget(t, keep=(m,))


# ---------------------------------------------------------------- aux Kalman
class AuxChain:
    def __init__(self, tg: OTarget, x0, delta):
        self.tg = tg
        self.c = Chain()
        self.x0 = _f64(x0)
        _check(lib().ao_init_chain(C.byref(tg.raw), _p(self.x0), delta, C.byref(self.c)), "init")

    def __del__(self):
        try:
            lib().ao_chain_free(C.byref(self.c))
        except Exception:
            pass

    @property
    def x(self):
        return np.ctypeslib.as_array(self.c.x, shape=(self.tg.T + 1, self.tg.dx)).copy()

    @property
    def grad_gen(self):
        return np.ctypeslib.as_array(self.c.grad_gen, shape=(self.tg.T + 1, self.tg.dx)).copy()

    def step(self, rng: Stream, backend=0, parallel_filter=0, zeroth_order=0):
        lib().ao_kernel_step(C.byref(self.tg.raw), C.byref(self.c), rng, backend,
                             parallel_filter, zeroth_order)

    def adapt(self, target_rate):
        lib().ao_adapt_delta(C.byref(self.c), target_rate)


def gamma_move(tg: OTarget, x, gamma: float, step: float, s: Stream):
    """runner.cpp:61-85: RW-MH on log gamma; returns (new gamma, accepted)."""
    g = C.c_double(gamma)
    moved = lib().ao_gamma_move(C.byref(tg.raw), _p(_f64(x)), C.byref(g), step, s)
    return g.value, bool(moved)


def aux_model_filter(tg: OTarget, x, u, delta, zeroth_order=False):
    """build_aux_lgssm (auxk.cpp:56-118) then kalman_filter; returns (FilterResult, obs)."""
    x, u = _f64(x), _f64(u)
    m = LGSSM()
    obs = C.POINTER(C.c_double)()
    lib().ao_build_aux_lgssm.argtypes = [C.POINTER(Target), PD, PD, C.c_double, C.c_int, PD,
                                         C.POINTER(LGSSM), C.POINTER(PD)]
    _check(lib().ao_build_aux_lgssm(C.byref(tg.raw), _p(x), _p(u), delta, int(zeroth_order), None,
                                    C.byref(m), C.byref(obs)), "build_aux_lgssm")
    T, dy = m.T, m.dy
    ob = np.ctypeslib.as_array(obs, shape=((T + 1) * dy,)).copy().reshape(T + 1, dy)
    fr = FilterResult(T, m.dx)
    raw = fr.raw()
    _check(lib().ao_kalman_filter(C.byref(m), obs, C.byref(raw)), "kalman_filter")
    fr.log_marginal = raw.log_marginal
    return fr, ob


def sample_aux_obs(x, delta, it: Stream):
    x = _f64(x)
    u = np.zeros_like(x)
    lib().ao_sample_aux_obs(_p(x), x.shape[0] - 1, x.shape[1], delta, it, _p(u))
    return u


def mh_log_ratio(tg: OTarget, x, xp, u, delta, zeroth_order=False):
    x, xp, u = _f64(x), _f64(xp), _f64(u)
    st = C.c_int(0)
    v = lib().ao_mh_log_ratio(C.byref(tg.raw), _p(x), _p(xp), _p(u), delta, int(zeroth_order),
                              C.byref(st))
    _check(st.value, "mh_log_ratio")
    return v


class PGChain:
    def __init__(self, tg: OTarget, x0, delta):
        self.tg = tg
        self.p = PG()
        self.x0 = _f64(x0)
        lib().ao_init_pg(C.byref(tg.raw), _p(self.x0), delta, C.byref(self.p))

    def __del__(self):
        try:
            lib().ao_pg_free(C.byref(self.p))
        except Exception:
            pass

    @property
    def x(self):
        return np.ctypeslib.as_array(self.p.x, shape=(self.tg.T + 1, self.tg.dx)).copy()

    @property
    def keys(self):
        return np.ctypeslib.as_array(self.p.keys, shape=(self.tg.T + 1,)).copy()

    def step(self, N, rng: Stream, mode=1, trace=False):
        T = self.tg.T
        anc = np.zeros((T + 1, N), np.int32) if trace else None
        sel = np.zeros(T + 1, np.int32) if trace else None
        bad = C.c_int(-1)
        st = lib().ao_aux_pgibbs_step(
            C.byref(self.tg.raw), C.byref(self.p), N, rng, mode,
            anc.ctypes.data_as(PI) if trace else None,
            sel.ctypes.data_as(PI) if trace else None, C.byref(bad))
        if trace:
            return st, bad.value, anc, sel
        return st, bad.value

    def adapt(self, target_rate):
        lib().ao_pg_adapt_delta(C.byref(self.p), target_rate)

    def step_pit(self, N, rng: Stream):
        sel = np.zeros(self.tg.T + 1, np.int32)
        bad = C.c_int(-1)
        st = lib().ao_pit_pgibbs_step(C.byref(self.tg.raw), C.byref(self.p), N, rng,
                                      sel.ctypes.data_as(PI), C.byref(bad))
        return st, bad.value, sel


def pit_csmc_marginals(tg: OTarget, u, delta, particles):
    u, particles = _f64(u), _f64(particles)
    T1, N = particles.shape[0], particles.shape[1]
    marg = np.zeros((T1, N))
    _check(lib().ao_pit_csmc_marginals(C.byref(tg.raw), _p(u), delta, _p(particles), N,
                                       _p(marg)), "pit_csmc_marginals")
    return marg


# ---------------------------------------------------------------- grid HMM oracle
def _logsumexp(v, axis=None):
    m = np.max(v, axis=axis, keepdims=True)
    m = np.where(np.isfinite(m), m, 0.0)
    return np.squeeze(m, axis=axis) + np.log(np.sum(np.exp(v - m), axis=axis))


def grid_hmm_posterior(tg: OTarget, lo: float, hi: float, n: int):
    """bench::grid_hmm_posterior (grid_hmm.cpp:17-97): smoothing marginals of a
    1-d target with linear dynamics on an equispaced midpoint grid, exact HMM
    forward-backward in log space.  Returns (points, marginals, mean, var, log_evidence)."""
    a = tg.arrays()
    if a["dx"] != 1 or not a["linear"]:
        raise ValueError("grid_hmm_posterior: 1-d linear-dynamics targets only")
    T = tg.T
    h = (hi - lo) / n
    logh = np.log(h)
    pts = lo + (np.arange(n) + 0.5) * h
    lpot = np.array([[tg.log_pot(t, [p]) for p in pts] for t in range(T + 1)])
    m0, p0 = a["m0"][0], a["P0"][0]
    nF = a["nF"]

    def lm(t):  # lm[i, j] = log p(x_{t+1} = pts[j] | x_t = pts[i]) (grid_hmm.cpp:38-47)
        k = t if nF > 1 else 0
        f, b, q = a["F"][k], a["b"][k], a["Q"][k]
        pred = f * pts + b
        return -0.5 * np.log(2.0 * np.pi * q) - (pts[None, :] - pred[:, None]) ** 2 / (2.0 * q)

    la = np.zeros((T + 1, n))
    lb = np.zeros((T + 1, n))
    la[0] = -0.5 * np.log(2.0 * np.pi * p0) - (pts - m0) ** 2 / (2.0 * p0) + lpot[0] + logh
    for t in range(T):
        la[t + 1] = _logsumexp(la[t][:, None] + lm(t), axis=0) + lpot[t + 1] + logh
    log_ev = float(_logsumexp(la[T]))
    for t in range(T - 1, -1, -1):
        lb[t] = _logsumexp(lm(t) + (lpot[t + 1] + lb[t + 1])[None, :], axis=1) + logh
    lg = la + lb
    lg -= _logsumexp(lg, axis=1)[:, None]
    marg = np.exp(lg)
    mean = marg @ pts
    var = marg @ (pts ** 2) - mean ** 2
    return pts, marg, mean, var, log_ev
