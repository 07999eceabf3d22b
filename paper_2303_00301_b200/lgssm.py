"""Linear-Gaussian state-space models on B200 — mirror of auxmc::lgssm
(lgssm.hpp:19-91) and auxmc::pit (pit.hpp:16-87), batched.

Arrays are torch float64 CUDA tensors, row-major.  A `Model` holds one
parameter set (per-step arrays or broadcast copies, lgssm.hpp:34-40); the
batched calls run many observation sequences or many paths against it.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


def _dev(x, device="cuda"):
    return torch.as_tensor(np.asarray(x, dtype=np.float64) if not torch.is_tensor(x) else x,
                           dtype=torch.float64).to(device).contiguous()


def _ptr(t):
    return None if t is None else t.data_ptr()


def _stream(device=None):
    return torch.cuda.current_stream(device).cuda_stream


class Model:
    """lgssm::Model (lgssm.hpp:19-49): x_{t+1} = F_t x_t + b_t + N(0,Q_t),
    y_t = H_t x_t + c_t + N(0,R_t) where observed.  Counts of F,b,Q are 1 or T;
    of H,c,R 1 or T+1.  Symmetrization of P0/Q/R happens inside the kernels."""

    def __init__(self, T, m0, P0, F, b, Q, H, c, R, obs_mask=None, device="cuda"):
        self.T = int(T)
        self.m0 = _dev(m0, device).reshape(-1)
        self.dx = self.m0.shape[0]
        dx = self.dx
        self.P0 = _dev(P0, device).reshape(dx, dx)
        self.F = _dev(F, device).reshape(-1, dx, dx)
        self.b = _dev(b, device).reshape(-1, dx)
        self.Q = _dev(Q, device).reshape(-1, dx, dx)
        H = _dev(H, device)
        self.dy = H.shape[-2] if H.numel() else 0
        self.H = H.reshape(-1, self.dy, dx)
        self.c = _dev(c, device).reshape(-1, self.dy)
        self.R = _dev(R, device).reshape(-1, self.dy, self.dy)
        self.mask = None if obs_mask is None else torch.as_tensor(
            np.asarray(obs_mask, dtype=np.uint8)).to(device)
        self.device = device
        for name, n, want in (("F", self.F.shape[0], self.T), ("b", self.b.shape[0], self.T),
                              ("Q", self.Q.shape[0], self.T), ("H", self.H.shape[0], self.T + 1),
                              ("c", self.c.shape[0], self.T + 1),
                              ("R", self.R.shape[0], self.T + 1)):
            if not (n == want or n == 1 or (want == 0 and n <= 1)):
                raise ValueError(f"Model: {name} count {n} (want 1 or {want})")

    @staticmethod
    def homogeneous(T, m0, P0, F, b, Q, H, c, R, obs_mask=None, device="cuda"):
        return Model(T, m0, P0, [np.asarray(F)], [np.asarray(b)], [np.asarray(Q)],
                     [np.asarray(H)], [np.asarray(c)], [np.asarray(R)], obs_mask, device)

    def horizon(self):
        return self.T

    def raw(self) -> _lib.Lgssm:
        m = _lib.Lgssm()
        m.T, m.dx, m.dy = self.T, self.dx, self.dy
        m.m0, m.P0 = _ptr(self.m0), _ptr(self.P0)
        m.F, m.nF = _ptr(self.F), self.F.shape[0]
        m.b, m.nb = _ptr(self.b), self.b.shape[0]
        m.Q, m.nQ = _ptr(self.Q), self.Q.shape[0]
        m.H, m.nH = _ptr(self.H), self.H.shape[0]
        m.c, m.nc = _ptr(self.c), self.c.shape[0]
        m.R, m.nR = _ptr(self.R), self.R.shape[0]
        m.mask = _ptr(self.mask)
        return m


@dataclass
class FilterResult:
    """lgssm::FilterResult (lgssm.hpp:51-55), batched over B sequences."""
    pred_mean: torch.Tensor   # [B, T+1, dx]
    pred_cov: torch.Tensor    # [B, T+1, dx, dx]
    filt_mean: torch.Tensor
    filt_cov: torch.Tensor
    log_marginal: torch.Tensor  # [B]
    status: torch.Tensor        # [B] int32

    @staticmethod
    def empty(B, T, dx, device="cuda"):
        z = lambda *s: torch.zeros(*s, dtype=torch.float64, device=device)
        return FilterResult(z(B, T + 1, dx), z(B, T + 1, dx, dx), z(B, T + 1, dx),
                            z(B, T + 1, dx, dx), z(B),
                            torch.zeros(B, dtype=torch.int32, device=device))

    def raw(self) -> _lib.FilterResult:
        f = _lib.FilterResult()
        f.pred_mean, f.pred_cov = _ptr(self.pred_mean), _ptr(self.pred_cov)
        f.filt_mean, f.filt_cov = _ptr(self.filt_mean), _ptr(self.filt_cov)
        f.log_marginal = _ptr(self.log_marginal)
        return f

    def select(self, b: int) -> "FilterResult":
        s = slice(b, b + 1)
        return FilterResult(self.pred_mean[s], self.pred_cov[s], self.filt_mean[s],
                            self.filt_cov[s], self.log_marginal[s], self.status[s])


def _filter(model: Model, obs, mode: int) -> FilterResult:
    obs = _dev(obs, model.device)
    if obs.dim() == 2:
        obs = obs.unsqueeze(0)
    B = obs.shape[0]
    if obs.shape[1:] != (model.T + 1, model.dy):
        raise ValueError("kalman_filter: observation array shape")
    fr = FilterResult.empty(B, model.T, model.dx, model.device)
    lib = _lib.load()
    mr = model.raw()
    ws_bytes = lib.auxmc_kalman_filter_workspace(C.byref(mr), B, mode)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=model.device)
    raw = fr.raw()
    _lib.check(lib.auxmc_kalman_filter(C.byref(mr), obs.data_ptr(), B, mode, C.byref(raw),
                                       fr.status.data_ptr(), ws.data_ptr(), ws_bytes,
                                       _stream()), "kalman_filter")
    fr._obs = obs
    return fr


def check_status(status: torch.Tensor, what: str):
    """Raise the reference's exception for a per-sequence / per-chain status array
    (FactorizationError, gauss.cpp:34, as AuxmcError code E_FACTOR).  Reads one int
    back from the device."""
    code = int(status.max()) if status.numel() else 0
    _lib.check(code, what)


def kalman_filter(model: Model, obs, check: bool = True) -> FilterResult:
    """lgssm::kalman_filter (lgssm.cpp:73-112) for obs [T+1, dy] or [B, T+1, dy].
    A covariance that fails the jitter ladder raises (check=True, the reference's
    behaviour) or is left in fr.status (check=False, per sequence)."""
    fr = _filter(model, obs, 0)
    if check:
        check_status(fr.status, "kalman_filter")
    return fr


def parallel_filter(model: Model, obs, check: bool = True) -> FilterResult:
    """pit::parallel_filter (pit.cpp:117-188): scan over filtering elements."""
    fr = _filter(model, obs, 1)
    if check:
        check_status(fr.status, "parallel_filter")
    return fr


class Noise:
    """NoiseSource analogue (rng.hpp:123-137): stream keys or pre-drawn arrays."""

    def __init__(self, keys=None, terminal=None, backward=None, bridge=None):
        self.keys = keys
        self.terminal = terminal
        self.backward = backward
        self.bridge = bridge

    @staticmethod
    def stream(keys: torch.Tensor) -> "Noise":
        return Noise(keys=keys.contiguous())

    @staticmethod
    def predrawn(terminal, backward, bridge=None, device="cuda") -> "Noise":
        return Noise(terminal=_dev(terminal, device), backward=_dev(backward, device),
                     bridge=None if bridge is None else _dev(bridge, device))

    @property
    def B(self):
        return self.keys.shape[0] if self.keys is not None else self.terminal.shape[0]

    def raw(self) -> _lib.Noise:
        n = _lib.Noise()
        if self.keys is not None:
            n.kind = _lib.NOISE_STREAM
            n.keys = _ptr(self.keys)
        else:
            n.kind = _lib.NOISE_PREDRAWN
            n.terminal = _ptr(self.terminal)
            n.backward = _ptr(self.backward)
            n.bridge = _ptr(self.bridge)
            n.n_bridge = 0 if self.bridge is None else self.bridge.shape[1]
        return n


class PathSampler:
    """Reusable launcher for pathwise draws (holds the workspace); the batched
    form of lgssm::backward_sample / pit::prefix_sample / pit::dnc_sample."""

    def __init__(self, model: Model, B: int, sampler: int, fr_shared: bool = True):
        self.model, self.B, self.sampler, self.fr_shared = model, B, sampler, fr_shared
        lib = _lib.load()
        self._mr = model.raw()
        self.ws_bytes = lib.auxmc_sample_paths_workspace(C.byref(self._mr), int(fr_shared), B,
                                                         sampler)
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=model.device)
        self.status = torch.zeros(B, dtype=torch.int32, device=model.device)

    def __call__(self, fr: FilterResult, noise: Noise, out: torch.Tensor = None,
                 stream=None, check: bool = False) -> torch.Tensor:
        """Draw the B paths.  self.status is reset every call and holds, per path,
        AUXMC_OK or AUXMC_E_FACTOR (a backward covariance / DnC bridge that failed the
        jitter ladder: that path is invalid).  check=True raises like the reference
        (one device read); hot loops keep check=False and call check_status()."""
        m = self.model
        if out is None:
            out = torch.empty((self.B, m.T + 1, m.dx), dtype=torch.float64, device=m.device)
        st = stream if stream is not None else _stream()
        fr_raw, nz = fr.raw(), noise.raw()
        _lib.check(_lib.load().auxmc_sample_paths(
            C.byref(self._mr), C.byref(fr_raw), int(self.fr_shared), C.byref(nz), self.B,
            self.sampler, out.data_ptr(), self.status.data_ptr(), self.ws.data_ptr(),
            self.ws_bytes, st), "sample_paths")
        if check:
            self.check_status()
        return out

    def check_status(self):
        check_status(self.status, "sample_paths")


class HostPipeline:
    """Pathwise draws for B chains from pinned HOST buffers with copy/compute overlap.

    The shared filter result is copied once per call; chains go in `chunks` equal
    chunks, and chunk i's host-to-device copy, chunk i-1's draw and chunk i-2's
    device-to-host copy run on three streams (double-buffered device staging), so
    the two PCIe directions overlap each other and the kernels.  Same draws as one
    PathSampler call over all B chains (chain c keeps its noise rows)."""

    def __init__(self, model: Model, B: int, sampler: int, chunks: int = 8):
        if B % chunks:
            raise ValueError("HostPipeline: chunks must divide the chain count")
        self.model, self.B, self.sampler, self.chunks = model, B, sampler, chunks
        self.Bc = B // chunks
        self.ps = PathSampler(model, self.Bc, sampler, True)
        self.s_in, self.s_run, self.s_out = (torch.cuda.Stream(model.device) for _ in range(3))
        self._buf = None
        self._fail = torch.zeros((), dtype=torch.int32, device=model.device)

    def _alloc(self, noise: Noise, fr: FilterResult):
        m, dev, Bc = self.model, self.model.device, self.Bc
        def like(t, rows):
            return torch.empty((rows,) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
        bufs = []
        for _ in range(2):
            b = {"out": torch.empty((Bc, m.T + 1, m.dx), dtype=torch.float64, device=dev)}
            for k in ("keys", "terminal", "backward", "bridge"):
                v = getattr(noise, k)
                b[k] = None if v is None else like(v, Bc)
            bufs.append(b)
        self._fr = FilterResult(*(torch.empty_like(t, device=dev) for t in
                                  (fr.pred_mean, fr.pred_cov, fr.filt_mean, fr.filt_cov,
                                   fr.log_marginal)), torch.zeros(1, dtype=torch.int32,
                                                                  device=dev))
        self._buf = bufs

    def __call__(self, fr_host: FilterResult, noise_host: Noise, out_host: torch.Tensor):
        if self._buf is None:
            self._alloc(noise_host, fr_host)
        main = torch.cuda.current_stream(self.model.device)
        ev = {k: [torch.cuda.Event() for _ in range(2)] for k in ("in", "run", "out")}
        self.s_in.wait_stream(main)
        with torch.cuda.stream(self.s_in):  # shared filter result, once
            for d, h in ((self._fr.pred_mean, fr_host.pred_mean), (self._fr.pred_cov,
                         fr_host.pred_cov), (self._fr.filt_mean, fr_host.filt_mean),
                         (self._fr.filt_cov, fr_host.filt_cov),
                         (self._fr.log_marginal, fr_host.log_marginal)):
                d.copy_(h, non_blocking=True)
        fr_ready = torch.cuda.Event()
        fr_ready.record(self.s_in)
        self.s_run.wait_event(fr_ready)
        with torch.cuda.stream(self.s_run):
            self._fail.zero_()
        for i in range(self.chunks):
            j, b = i % 2, self._buf[i % 2]
            sl = slice(i * self.Bc, (i + 1) * self.Bc)
            if i >= 2:
                self.s_in.wait_event(ev["run"][j])   # staging j consumed by draw i-2
                self.s_run.wait_event(ev["out"][j])  # output j drained by copy i-2
            with torch.cuda.stream(self.s_in):
                for k in ("keys", "terminal", "backward", "bridge"):
                    if b[k] is not None:
                        b[k].copy_(getattr(noise_host, k)[sl], non_blocking=True)
                ev["in"][j].record(self.s_in)
            self.s_run.wait_event(ev["in"][j])
            with torch.cuda.stream(self.s_run):
                nz = Noise(keys=b["keys"], terminal=b["terminal"], backward=b["backward"],
                           bridge=b["bridge"])
                self.ps(self._fr, nz, b["out"])
                torch.maximum(self._fail, self.ps.status.amax(), out=self._fail)
                ev["run"][j].record(self.s_run)
            self.s_out.wait_event(ev["run"][j])
            with torch.cuda.stream(self.s_out):
                out_host[sl].copy_(b["out"], non_blocking=True)
                ev["out"][j].record(self.s_out)
        main.wait_stream(self.s_out)
        main.wait_stream(self.s_run)
        return out_host

    def check_status(self):
        """Raise if any chunk of the last pass had a factorization failure."""
        _lib.check(int(self._fail), "HostPipeline")


def _sample(model, fr, noise, sampler):
    B = noise.B
    shared = fr.filt_mean.shape[0] == 1
    return PathSampler(model, B, sampler, shared)(fr, noise, check=True)


def backward_sample(model: Model, fr: FilterResult, noise: Noise) -> torch.Tensor:
    """lgssm::backward_sample (lgssm.cpp:151-177), one path per noise row."""
    return _sample(model, fr, noise, _lib.SAMPLER_SEQ)


def path_logpdf(model: Model, obs, traj, fr: FilterResult) -> torch.Tensor:
    """lgssm::path_logpdf (lgssm.cpp:179-199) for traj [B, T+1, dx]."""
    obs = _dev(obs, model.device)
    if obs.dim() == 2:
        obs = obs.unsqueeze(0)
    traj = _dev(traj, model.device)
    if traj.dim() == 2:
        traj = traj.unsqueeze(0)
    B = traj.shape[0]
    out = torch.empty(B, dtype=torch.float64, device=model.device)
    status = torch.zeros(B, dtype=torch.int32, device=model.device)
    mr, fr_raw = model.raw(), fr.raw()
    _lib.check(_lib.load().auxmc_path_logpdf(
        C.byref(mr), obs.data_ptr(), int(obs.shape[0] == 1), traj.data_ptr(), C.byref(fr_raw),
        int(fr.filt_mean.shape[0] == 1), B, out.data_ptr(), status.data_ptr(), _stream()),
        "path_logpdf")
    check_status(status, "path_logpdf")
    return out


def rts_smoother(model: Model, fr: FilterResult):
    """lgssm::rts_smoother (lgssm.cpp:114-127): smoothed marginals
    (mean [B, T+1, dx], cov [B, T+1, dx, dx]) for every filter result in fr."""
    B = fr.filt_mean.shape[0]
    dev = model.device
    mean = torch.empty((B, model.T + 1, model.dx), dtype=torch.float64, device=dev)
    cov = torch.empty((B, model.T + 1, model.dx, model.dx), dtype=torch.float64, device=dev)
    status = torch.zeros(B, dtype=torch.int32, device=dev)
    lib = _lib.load()
    mr, fr_raw = model.raw(), fr.raw()
    n = lib.auxmc_rts_smoother_workspace(C.byref(mr), B)
    ws = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    _lib.check(lib.auxmc_rts_smoother(C.byref(mr), C.byref(fr_raw), B, mean.data_ptr(),
                                      cov.data_ptr(), status.data_ptr(), ws.data_ptr(), n,
                                      _stream()), "rts_smoother")
    _lib.check(int(status.max()), "rts_smoother")
    return mean, cov
