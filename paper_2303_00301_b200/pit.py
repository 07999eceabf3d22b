"""Parallel-in-time samplers and filter — mirror of auxmc::pit (pit.hpp:16-87)."""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from .lgssm import FilterResult, Model, Noise, PathSampler, parallel_filter  # noqa: F401


class Sampler:
    kSequential = _lib.SAMPLER_SEQ
    kPrefix = _lib.SAMPLER_PREFIX
    kDnc = _lib.SAMPLER_DNC


def prefix_sample(model: Model, fr: FilterResult, noise: Noise) -> torch.Tensor:
    """pit::prefix_sample (pit.cpp:78-115): suffix scan of realized elements."""
    shared = fr.filt_mean.shape[0] == 1
    return PathSampler(model, noise.B, _lib.SAMPLER_PREFIX, shared)(fr, noise, check=True)


def dnc_sample(model: Model, fr: FilterResult, noise: Noise) -> torch.Tensor:
    """pit::dnc_sample (pit.cpp:192-301): bridges over the fixed segment tree."""
    shared = fr.filt_mean.shape[0] == 1
    return PathSampler(model, noise.B, _lib.SAMPLER_DNC, shared)(fr, noise, check=True)


def dnc_bridge_count(T: int) -> int:
    return _lib.load().auxmc_dnc_bridge_count(T)


def extract_affine_law(which: int, model: Model, fr: FilterResult):
    """pit::extract_affine_law (pit.cpp:303-332) on the device: the exact law
    N(mean [n], cov [n, n]) of sampler `which` over the flat path index t*dx + j,
    from the zero noise and every basis noise vector in one pre-drawn batch."""
    lib = _lib.load()
    n = (model.T + 1) * model.dx
    dev = model.device
    mean = torch.empty(n, dtype=torch.float64, device=dev)
    cov = torch.empty((n, n), dtype=torch.float64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    mr, fr_raw = model.raw(), fr.raw()
    nb = lib.auxmc_affine_law_workspace(C.byref(mr), int(which))
    ws = torch.empty(max(nb, 1), dtype=torch.uint8, device=dev)
    _lib.check(lib.auxmc_affine_law(C.byref(mr), C.byref(fr_raw), int(which), mean.data_ptr(),
                                    cov.data_ptr(), status.data_ptr(), ws.data_ptr(), nb,
                                    torch.cuda.current_stream(dev).cuda_stream),
               "extract_affine_law")
    _lib.check(int(status[0]), "extract_affine_law")
    return mean, cov
