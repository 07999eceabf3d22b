"""Counter-based streams (rng.hpp:35-118) — host side, via libauxmc_b200.

`RngStream` has the reference's value semantics: `from_seed`, `derive(label,
index)`, `next_uniform`, `next_normal`, `normal_vec`, `next_key`, `from_key`.
Batched device keys for many chains come from `chain_keys`.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib

kBackwardNoise, kTerminalDraw, kAuxObs, kDncBridge, kMhAccept = 1, 2, 3, 4, 5
kIteration, kChain, kStep, kParticle, kResample = 6, 7, 8, 9, 10
kTerminalIndex, kBackwardIndex, kPmKey, kSimulate, kParam = 11, 12, 13, 14, 15


class RngStream:
    __slots__ = ("key", "counter")

    def __init__(self, key: int = 0, counter: int = 0):
        self.key = int(key)
        self.counter = int(counter)

    @staticmethod
    def from_seed(seed: int) -> "RngStream":
        return RngStream(_lib.load().auxmc_rng_from_seed(seed))

    @staticmethod
    def from_key(key: int) -> "RngStream":
        return RngStream(key)

    def derive(self, label: int, index: int) -> "RngStream":
        return RngStream(_lib.load().auxmc_rng_derive(self.key, label, index))

    def next_uniform(self) -> float:
        v = _lib.load().auxmc_rng_uniform(self.key, self.counter)
        self.counter += 1
        return v

    def next_normal(self) -> float:
        v = _lib.load().auxmc_rng_normal(self.key, self.counter)
        self.counter += 1
        return v

    def normal_vec(self, d: int) -> np.ndarray:
        return np.array([self.next_normal() for _ in range(d)])

    def __repr__(self):
        return f"RngStream(key=0x{self.key:016x}, counter={self.counter})"


def chain_keys(seed: int, n_chains: int, first: int = 0, device="cuda") -> torch.Tensor:
    """Chain roots from_seed(seed).derive(kChain, c) for c in [first, first+n) as uint64
    (int64 storage), the batched form of runner.cpp:132."""
    root = RngStream.from_seed(seed)
    keys = [root.derive(kChain, c).key for c in range(first, first + n_chains)]
    arr = np.array(keys, dtype=np.uint64).view(np.int64)
    return torch.from_numpy(arr).to(device)


def iteration_keys(root_keys: torch.Tensor, it: int) -> torch.Tensor:
    """it = root.derive(kIteration, iter) per chain (auxk.cpp:132)."""
    lib = _lib.load()
    ks = root_keys.cpu().numpy().view(np.uint64)
    out = np.array([lib.auxmc_rng_derive(int(k), kIteration, it) for k in ks], dtype=np.uint64)
    return torch.from_numpy(out.view(np.int64)).to(root_keys.device)


def normals(keys: torch.Tensor, label: int, index0: int, n_index: int, dim: int,
            stream=None) -> torch.Tensor:
    """Device draws out[b, i, :] = keys[b].derive(label, index0+i).normal_vec(dim)."""
    B = keys.shape[0]
    out = torch.empty((B, n_index, dim), dtype=torch.float64, device=keys.device)
    st = stream if stream is not None else torch.cuda.current_stream(keys.device).cuda_stream
    _lib.check(_lib.load().auxmc_rng_normals(keys.data_ptr(), B, label, index0, n_index, dim,
                                             out.data_ptr(), st), "auxmc_rng_normals")
    return out
