"""Auxiliary Kalman sampler on B200 — mirror of auxmc::auxk (target.hpp:34-93,
auxk.hpp:15-79), batched over chains.

`GenSSMTarget` is the device descriptor of a target over x_{0:T}; model
closures of the reference become device functors selected by kind.
`AuxChains` holds C chain states (AuxChainState, auxk.hpp:50-57) in HBM and
advances them with `kernel_step` (auxk.cpp:130-198), `adapt_delta`
(auxk.cpp:213-218) and `init_chain` (auxk.cpp:120-128).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .bench_models import KIND, ModelSpec, obs_dim, latent_dim, simulate, synth_mats, target_params
from .rng import chain_keys


class Backend:
    kSequential = 0
    kPrefix = 1
    kDnc = 2


def _t(a, device, dtype=torch.float64):
    host = np.array(a, dtype=np.float64 if dtype == torch.float64 else np.uint8, copy=True)
    return torch.from_numpy(host).to(device=device, dtype=dtype).contiguous()


def _unit_selection(H, R) -> bool:
    """Each exact row observes one state component with unit gain (distinct components)
    under a diagonal positive R_e: the fused direct-observation filter applies."""
    H = np.asarray(H, np.float64)
    R = np.asarray(R, np.float64).reshape(H.shape[0], H.shape[0])
    nz = H != 0.0
    if not (nz.sum(axis=1) == 1).all() or not (H[nz] == 1.0).all():
        return False
    cols = nz.argmax(axis=1)
    if len(set(cols.tolist())) != len(cols):
        return False
    return bool((R == np.diag(np.diag(R))).all() and (np.diag(R) > 0).all())


class GenSSMTarget:
    """Device target: linear or tractable dynamics × exact / generic potentials."""

    def __init__(self, kind, T, dx, m0, P0, Q, F=None, b=None, *, linear=True, eH=None, ec=None,
                 eR=None, ey=None, emask=None, data=None, gmask=None, gH=None, gc=None, gR=None,
                 params=None, device="cuda"):
        self.kind = KIND[kind] if isinstance(kind, str) else int(kind)
        self.T, self.dx, self.device = int(T), int(dx), device
        d = self.dx
        self.linear = bool(linear)
        self.m0 = _t(m0, device).reshape(d)
        self.P0 = _t(P0, device).reshape(d, d)
        self.Q = _t(Q, device).reshape(-1, d, d)
        self.nF = self.Q.shape[0]
        self.F = None if F is None else _t(F, device).reshape(-1, d, d)
        self.b = None if b is None else _t(b, device).reshape(-1, d)
        if self.linear and (self.F is None or self.b is None):
            raise ValueError("linear target needs F and b")
        T1 = self.T + 1
        self.q = 0 if eH is None else np.asarray(eH).shape[-2]
        self.ne = 1
        if eH is not None:
            eHn = np.asarray(eH, dtype=np.float64).reshape(-1, self.q, d)
            self.ne = eHn.shape[0]
            self.eH = _t(eHn, device)
            self.ec = _t(np.asarray(ec, np.float64).reshape(self.ne, self.q), device)
            self.eR = _t(np.asarray(eR, np.float64).reshape(self.ne, self.q, self.q), device)
            self.ey = _t(np.asarray(ey, np.float64).reshape(T1, self.q), device)
        else:
            self.eH = self.ec = self.eR = self.ey = None
        em = np.ones(T1, np.uint8) if emask is None else np.asarray(emask, np.uint8)
        if self.q == 0:
            em = np.zeros(T1, np.uint8)
        self.emask_host = em
        self.emask = _t(em, device, torch.uint8)
        self.exact_tv = int(self.q > 0 and (self.ne > 1 or (em.min() != em.max())))
        self.exact_sel = int(self.q == 0 or (self.ne == 1 and _unit_selection(eHn[0], eR)))
        self.data = None if data is None else _t(data, device).reshape(T1, -1)
        self.ydim = 0 if data is None else self.data.shape[1]
        gm = np.zeros(T1, np.uint8) if gmask is None else np.asarray(gmask, np.uint8)
        self.gmask = _t(gm, device, torch.uint8)
        self.gH = None if gH is None else _t(gH, device)
        self.gc = None if gc is None else _t(gc, device)
        self.gR = None if gR is None else _t(gR, device)
        if self.kind == KIND["gauss-generic"]:
            self.ne = self.gH.reshape(-1, self.ydim, d).shape[0]
        self.params = dict(lz_sigma=10.0, lz_rho=28.0, lz_beta=8.0 / 3.0, lz_h=0.01, l96_F=8.0,
                           l96_h=0.01)
        if params:
            self.params.update(params)

    def horizon(self):
        return self.T

    def max_exact_rows(self):
        return self.q

    def raw(self) -> _lib.Target:
        r = _lib.Target()
        p = lambda t: None if t is None else t.data_ptr()
        r.kind, r.T, r.dx, r.ydim, r.linear = self.kind, self.T, self.dx, self.ydim, int(self.linear)
        r.m0, r.P0, r.F, r.b, r.Q, r.nF = p(self.m0), p(self.P0), p(self.F), p(self.b), p(self.Q), self.nF
        r.q, r.ne, r.exact_tv = self.q, self.ne, self.exact_tv
        r.exact_sel = self.exact_sel
        r.eH, r.ec, r.eR, r.ey = p(self.eH), p(self.ec), p(self.eR), p(self.ey)
        r.emask, r.data, r.gmask = p(self.emask), p(self.data), p(self.gmask)
        r.gH, r.gc, r.gR = p(self.gH), p(self.gc), p(self.gR)
        for k, v in self.params.items():
            setattr(r, k, v)
        return r

    def log_gamma(self, traj) -> torch.Tensor:
        """target.log_gamma (target.cpp:100-108) for [B, T+1, dx] paths."""
        traj = torch.as_tensor(traj, dtype=torch.float64, device=self.device)
        if traj.dim() == 2:
            traj = traj.unsqueeze(0)
        traj = traj.contiguous()
        B = traj.shape[0]
        out = torch.empty(B, dtype=torch.float64, device=self.device)
        st = torch.zeros(B, dtype=torch.int32, device=self.device)
        r = self.raw()
        _lib.check(_lib.load().auxmc_log_gamma(C.byref(r), traj.data_ptr(), B, out.data_ptr(),
                                               st.data_ptr(), torch.cuda.current_stream().cuda_stream),
                   "log_gamma")
        return out

    # ---- constructors
    @staticmethod
    def linear_exact(m, obs, device="cuda"):
        """testutil.hpp:88-108: LGSSM posterior with exact Gaussian potentials.
        `m` is any object with numpy fields T, m0, P0, F, b, Q, H, c, R, mask."""
        T = m.T
        mask = np.ones(T + 1, np.uint8) if m.mask is None else np.asarray(m.mask, np.uint8)
        nd = max(m.F.shape[0], m.b.shape[0], m.Q.shape[0])
        bc = lambda a: np.broadcast_to(a, (nd,) + a.shape[1:]) if a.shape[0] == 1 else a
        ne = max(m.H.shape[0], m.c.shape[0], m.R.shape[0])
        bo = lambda a: np.broadcast_to(a, (ne,) + a.shape[1:]) if a.shape[0] == 1 else a
        return GenSSMTarget("lgssm-synthetic", T, m.dx, m.m0, m.P0, bc(m.Q), bc(m.F), bc(m.b),
                            eH=bo(m.H), ec=bo(m.c), eR=bo(m.R), ey=obs, emask=mask, device=device)

    @staticmethod
    def test_kind(name, T, device="cuda"):
        """Test-only targets reaching the reference's failure semantics (auxmc_gpu.h
        AUXMC_KIND_TEST_*): 1-d linear dynamics m0 = 0, P0 = 0.04, F = 0.5, b = 0,
        Q = 0.04 with the generic potentials of test_target_auxk.cpp:374-414 ("test-abort",
        "test-support") and test_fkpg.cpp:447-465 ("test-collapse")."""
        if name not in ("test-abort", "test-support", "test-collapse"):
            raise ValueError(name)
        return GenSSMTarget(name, T, 1, [0.0], [[0.04]], [[[0.04]]], [[[0.5]]], [[0.0]],
                            gmask=np.ones(T + 1, np.uint8), device=device)

    @staticmethod
    def linear_generic(m, obs, device="cuda"):
        """testutil.hpp:112-140: same law, Gaussian potentials in generic form."""
        T = m.T
        mask = np.ones(T + 1, np.uint8) if m.mask is None else np.asarray(m.mask, np.uint8)
        nd = max(m.F.shape[0], m.b.shape[0], m.Q.shape[0])
        bc = lambda a: np.broadcast_to(a, (nd,) + a.shape[1:]) if a.shape[0] == 1 else a
        ne = max(m.H.shape[0], m.c.shape[0], m.R.shape[0])
        bo = lambda a: np.broadcast_to(a, (ne,) + a.shape[1:]) if a.shape[0] == 1 else a
        return GenSSMTarget("gauss-generic", T, m.dx, m.m0, m.P0, bc(m.Q), bc(m.F), bc(m.b),
                            data=obs, gmask=mask, gH=bo(m.H), gc=bo(m.c), gR=bo(m.R),
                            device=device)


def make_target(spec: ModelSpec, data, device="cuda") -> GenSSMTarget:
    """bench::make_target (models.cpp:240-336) as a device target."""
    dx, dy, T = latent_dim(spec), obs_dim(spec), spec.T
    data = np.asarray(data, np.float64).reshape(T + 1, max(dy, 0))
    tp = target_params(spec)
    kind = spec.kind
    if kind == "lgssm-synthetic":
        mm = synth_mats(spec)
        return GenSSMTarget(kind, T, dx, tp["m0"], tp["P0"], tp["Q"], tp["F"], tp["b"],
                            eH=mm["H"], ec=np.zeros(dy), eR=mm["R"], ey=data, device=device)
    if kind in ("stochvol", "spatio-temporal", "grid-1d-test"):
        return GenSSMTarget(kind, T, dx, tp["m0"], tp["P0"], tp["Q"], tp["F"], tp["b"],
                            data=data if dy > 0 else None, gmask=np.ones(T + 1, np.uint8),
                            device=device)
    if kind in ("diffusion-smoothing", "lorenz96"):
        q = dy
        H = np.zeros((q, dx))
        for k in range(q):
            H[k, 2 * k] = 1.0
        ov = spec.lz_obs_var if kind == "diffusion-smoothing" else spec.l96_obs_var
        return GenSSMTarget(kind, T, dx, tp["m0"], tp["P0"], tp["Q"], linear=False, eH=H,
                            ec=np.zeros(q), eR=ov * np.eye(q), ey=data,
                            params=dict(lz_sigma=spec.lz_sigma, lz_rho=spec.lz_rho,
                                        lz_beta=spec.lz_beta, lz_h=spec.lz_h, l96_F=spec.l96_F,
                                        l96_h=spec.l96_h), device=device)
    raise ValueError(f"unknown model kind {kind}")


class AuxChains:
    """C chain states (AuxChainState, auxk.hpp:50-57) resident in HBM."""

    def __init__(self, target: GenSSMTarget, x0, delta, root_keys: torch.Tensor):
        dev = target.device
        self.target = target
        x0 = torch.as_tensor(x0, dtype=torch.float64, device=dev)
        Cn = root_keys.shape[0]
        if x0.dim() == 2:
            x0 = x0.unsqueeze(0).expand(Cn, -1, -1)
        self.C = Cn
        self.x = x0.contiguous().clone()
        self.delta = torch.full((Cn,), float(delta), dtype=torch.float64, device=dev) \
            if np.isscalar(delta) else torch.as_tensor(delta, dtype=torch.float64, device=dev).clone()
        self.log_gamma = torch.zeros(Cn, dtype=torch.float64, device=dev)
        self.grad_gen = torch.zeros_like(self.x)
        self.iter = torch.zeros(Cn, dtype=torch.int64, device=dev)
        self.stats = torch.zeros((Cn, 6), dtype=torch.float64, device=dev)  # 4 int64 + 2 double
        self.stats.view(torch.int64)[:, :4] = 0
        self.stats[:, 4] = 0.0
        self.root_keys = root_keys.contiguous()
        self._ws = None
        self._ws_key = None
        self.init()

    def raw(self) -> _lib.Chains:
        r = _lib.Chains()
        r.C = self.C
        r.x, r.delta, r.log_gamma = self.x.data_ptr(), self.delta.data_ptr(), self.log_gamma.data_ptr()
        r.grad_gen, r.iter, r.stats = self.grad_gen.data_ptr(), self.iter.data_ptr(), self.stats.data_ptr()
        r.root_keys = self.root_keys.data_ptr()
        return r

    def _workspace(self, nbytes):
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(nbytes, dtype=torch.uint8, device=self.target.device)
        return self._ws

    def init(self):
        """auxk::init_chain (auxk.cpp:120-128) for every chain."""
        tr, ch = self.target.raw(), self.raw()
        ws = self._workspace(64 << 20)
        _lib.check(_lib.load().auxmc_init_chains(C.byref(tr), C.byref(ch), ws.data_ptr(),
                                                 ws.numel(), torch.cuda.current_stream().cuda_stream),
                   "init_chains")

    def kernel_step(self, backend=Backend.kSequential, zeroth_order=False, parallel_filter=False,
                    stream=None):
        """auxk::kernel_step (auxk.cpp:130-198) for every chain; KernelOptions fields
        (auxk.hpp:34-39) as keyword arguments."""
        lib = _lib.load()
        tr, ch = self.target.raw(), self.raw()
        o = _lib.KernelOptions(int(backend), int(parallel_filter), int(zeroth_order))
        key = (int(backend), bool(zeroth_order), bool(parallel_filter))
        if self._ws_key != key:
            self._ws_bytes = lib.auxmc_aux_kernel_workspace(C.byref(tr), self.C, C.byref(o))
            self._ws_key = key
        ws = self._workspace(self._ws_bytes)
        _lib.check(lib.auxmc_aux_kernel_step(C.byref(tr), C.byref(ch), C.byref(o), ws.data_ptr(),
                                             ws.numel(), stream if stream is not None else
                                             torch.cuda.current_stream().cuda_stream),
                   "aux_kernel_step")

    def graph_step(self, backend=Backend.kSequential, zeroth_order=False, parallel_filter=False):
        """kernel_step replayed from a CUDA graph: the first call per option set
        captures the whole step (every kernel of auxk.cpp:130-198 for all chains,
        stream-ordered, workspace preallocated) and later calls are one graph
        launch.  Chain state is updated in place, iteration keys come from the
        device-side counters, so replays are bit-identical to eager steps."""
        lib = _lib.load()
        key = (int(backend), bool(zeroth_order), bool(parallel_filter))
        if not hasattr(self, "_graphs"):
            self._graphs = {}
        if key not in self._graphs:
            tr = self.target.raw()
            o = _lib.KernelOptions(*[int(k) for k in key])
            if self._ws_key != key:
                self._ws_bytes = lib.auxmc_aux_kernel_workspace(C.byref(tr), self.C, C.byref(o))
                self._ws_key = key
            self._workspace(self._ws_bytes)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            n0 = lib.auxmc_launch_count()
            with torch.cuda.graph(g, capture_error_mode="relaxed"):
                self.kernel_step(backend, zeroth_order, parallel_filter)
            self._graphs[key] = (g, lib.auxmc_launch_count() - n0)
        g, _ = self._graphs[key]
        g.replay()

    def graph_launches(self, backend=Backend.kSequential, zeroth_order=False,
                       parallel_filter=False):
        """Kernels in the captured step graph (0 before the first graph_step)."""
        key = (int(backend), bool(zeroth_order), bool(parallel_filter))
        return getattr(self, "_graphs", {}).get(key, (None, 0))[1]

    def adapt_delta(self, target_rate):
        ch = self.raw()
        _lib.check(_lib.load().auxmc_adapt_delta(C.byref(ch), float(target_rate),
                                                 torch.cuda.current_stream().cuda_stream),
                   "adapt_delta")

    # KernelStats view (auxk.hpp:41-48)
    @property
    def accepted(self):
        return self.stats.view(torch.int64)[:, 0]

    @property
    def rejected(self):
        return self.stats.view(torch.int64)[:, 1]

    @property
    def aborted(self):
        return self.stats.view(torch.int64)[:, 2]

    @property
    def nonfinite_gamma(self):
        return self.stats.view(torch.int64)[:, 3]

    @property
    def last_log_alpha(self):
        return self.stats[:, 4]

    @property
    def last_accept_prob(self):
        return self.stats[:, 5]


def init_chains(target: GenSSMTarget, x0, delta, seed: int, n_chains: int, first: int = 0):
    """Batched init_chain with chain roots from_seed(seed).derive(kChain, c) (runner.cpp:132)."""
    return AuxChains(target, x0, delta, chain_keys(seed, n_chains, first, target.device))


def gamma_move(target: GenSSMTarget, x, root_keys: torch.Tensor, iter: int, step: float,
               gamma) -> tuple[torch.Tensor, torch.Tensor]:
    """bench/runner.cpp:61-85 `gamma_move` for C chains: random-walk MH on log γ (the
    diffusion coefficient of a Lorenz target, Q = h γ² I) with a N(0, 1) prior on log γ,
    stream root.derive(kParam, iter) per chain.  `x` [C, T+1, dx] device paths, `gamma`
    a scalar or [C].  Returns (new γ [C], accepted [C] bool).  Like the reference, the
    caller rebuilds the target with the new γ (runner.cpp:162-167)."""
    x = torch.as_tensor(x, dtype=torch.float64, device=target.device)
    if x.dim() == 2:
        x = x.unsqueeze(0)
    x = x.contiguous()
    Cn = x.shape[0]
    if tuple(x.shape[1:]) != (target.T + 1, target.dx):
        raise ValueError(f"gamma_move: paths must be [C, {target.T + 1}, {target.dx}]")
    if not torch.is_tensor(root_keys) or root_keys.dtype not in (torch.int64, torch.uint64) \
            or root_keys.dim() != 1:
        raise ValueError("gamma_move: root_keys must be a 1-D int64/uint64 tensor")
    keys = root_keys.to(target.device).contiguous()
    if keys.shape[0] != Cn:
        raise ValueError("gamma_move: one root key per chain")
    g = torch.full((Cn,), float(gamma), dtype=torch.float64, device=target.device) \
        if np.isscalar(gamma) else torch.as_tensor(gamma, dtype=torch.float64,
                                                   device=target.device).reshape(-1).clone()
    if g.numel() != Cn:
        raise ValueError("gamma_move: gamma must be a scalar or one value per chain")
    moved = torch.zeros(Cn, dtype=torch.int32, device=target.device)
    r = target.raw()
    _lib.check(_lib.load().auxmc_gamma_move(C.byref(r), Cn, x.data_ptr(), keys.data_ptr(), int(iter),
                                            float(step), g.data_ptr(), moved.data_ptr(),
                                            torch.cuda.current_stream().cuda_stream),
               "gamma_move")
    return g, moved.bool()
