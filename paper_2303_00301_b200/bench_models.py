"""Bench models — mirror of auxmc::bench (bench/models.hpp:16-89).

ModelSpec fields, `simulate`, `synthetic_lgssm` and `make_target` with the
reference's names.  Data generation is host C++ inside libauxmc_b200
(host/models.cpp); targets are device descriptors consumed by the kernels.
Adds the Lorenz-96 model the benchmark configs name (kind "lorenz96").
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, fields

import numpy as np
import torch

from . import _lib

KIND = _lib.KIND


@dataclass
class ModelSpec:
    kind: str = "lgssm-synthetic"
    T: int = 50
    dx: int = 2
    dy: int = 1
    grid: int = 3
    data_seed: int = 1
    sv_mu: float = -1.0
    sv_phi: float = 0.9
    sv_sig2: float = 0.1
    sv_rho: float = 0.25
    lz_sigma: float = 10.0
    lz_rho: float = 28.0
    lz_beta: float = 8.0 / 3.0
    lz_h: float = 0.01
    lz_gamma: float = 2.0
    lz_obs_var: float = 1.0
    st_phi: float = 0.8
    st_kappa2: float = 1.0
    st_tau2: float = 0.3
    g1_phi: float = 0.8
    g1_q: float = 0.09
    g1_m0: float = 0.5
    g1_p0: float = 0.25
    l96_F: float = 8.0
    l96_h: float = 0.01
    l96_gamma: float = 1.0
    l96_obs_var: float = 1.0

    def raw(self) -> _lib.ModelSpec:
        s = _lib.ModelSpec()
        for f in fields(self):
            v = getattr(self, f.name)
            setattr(s, f.name, KIND[v] if f.name == "kind" else v)
        return s


def latent_dim(spec: ModelSpec) -> int:
    return _lib.load().auxmc_latent_dim(C.byref(spec.raw()))


def obs_dim(spec: ModelSpec) -> int:
    return _lib.load().auxmc_obs_dim(C.byref(spec.raw()))


def _pd(a):
    return a.ctypes.data_as(_lib.PD)


def simulate(spec: ModelSpec):
    """bench::simulate (models.cpp:162-238): (latent [T+1, dx], data [T+1, ydim])."""
    dx, dy = latent_dim(spec), obs_dim(spec)
    lat = np.zeros((spec.T + 1, dx))
    data = np.zeros((spec.T + 1, max(dy, 1)))
    _lib.check(_lib.load().auxmc_simulate(C.byref(spec.raw()), _pd(lat), _pd(data)), "simulate")
    return lat, data[:, :dy]


def synth_mats(spec: ModelSpec) -> dict:
    dx, dy = spec.dx, spec.dy
    out = dict(m0=np.zeros(dx), b=np.zeros(dx), P0=np.zeros((dx, dx)), F=np.zeros((dx, dx)),
               Q=np.zeros((dx, dx)), H=np.zeros((dy, dx)), R=np.zeros((dy, dy)))
    _lib.check(_lib.load().auxmc_synth_mats(
        C.byref(spec.raw()), _pd(out["m0"]), _pd(out["b"]), _pd(out["P0"]), _pd(out["F"]),
        _pd(out["Q"]), _pd(out["H"]), _pd(out["R"])), "synth_mats")
    return out


def synthetic_lgssm(spec: ModelSpec, device="cuda"):
    """bench::synthetic_lgssm (models.cpp:338-344)."""
    from .lgssm import Model
    m = synth_mats(spec)
    return Model.homogeneous(spec.T, m["m0"], m["P0"], m["F"], m["b"], m["Q"], m["H"],
                             np.zeros(spec.dy), m["R"], device=device)


def target_params(spec: ModelSpec) -> dict:
    dx = latent_dim(spec)
    out = dict(m0=np.zeros(dx), P0=np.zeros((dx, dx)), F=np.zeros((dx, dx)), b=np.zeros(dx),
               Q=np.zeros((dx, dx)))
    _lib.check(_lib.load().auxmc_target_params(
        C.byref(spec.raw()), _pd(out["m0"]), _pd(out["P0"]), _pd(out["F"]), _pd(out["b"]),
        _pd(out["Q"])), "target_params")
    return out
