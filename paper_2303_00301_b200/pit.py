"""Parallel-in-time samplers and filter — mirror of auxmc::pit (pit.hpp:16-87)."""
from __future__ import annotations

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
    return PathSampler(model, noise.B, _lib.SAMPLER_PREFIX, shared)(fr, noise)


def dnc_sample(model: Model, fr: FilterResult, noise: Noise) -> torch.Tensor:
    """pit::dnc_sample (pit.cpp:192-301): bridges over the fixed segment tree."""
    shared = fr.filt_mean.shape[0] == 1
    return PathSampler(model, noise.B, _lib.SAMPLER_DNC, shared)(fr, noise)


def dnc_bridge_count(T: int) -> int:
    return _lib.load().auxmc_dnc_bridge_count(T)
