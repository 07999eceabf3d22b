"""Auxiliary particle Gibbs on B200 — mirror of auxmc::fkpg (fkpg.hpp:61-109).

`PGChains` holds C particle-Gibbs states (PGState, fkpg.hpp:92-99) in HBM.
`aux_pgibbs_step` runs one sweep for every chain (fkpg.cpp:260-274) with the
proposal mode of PgOptions (prior, gradient or fully adapted, linearized at the
auxiliary observation; fkpg.cpp:154-185), in one of two variants:
  Variant.kReference — the reference conditional SMC (multinomial resampling,
                       backward index sampling; fkpg.cpp:44-152);
  Variant.kPit       — parallel-in-time cSMC with independent proposals
                       (gradient mode only: the lattice needs parent-free proposals).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .auxk import GenSSMTarget
from .rng import chain_keys


class ProposalMode:
    kPrior = 0
    kGradient = 1
    kFullyAdapted = 2


class Variant:
    kReference = 0
    kPit = 1


class PseudoMarginal:
    """Device pseudo-marginal estimators (auxmc_gpu.h AUXMC_PM_*): the reference's
    pm_potential (fkpg.cpp:233-250) with the estimators of its own tests."""
    kNone = 0
    kTwoPoint = 1   # exp(log g) * (U(key) < 0.5 ? 0.5 : 1.5), acceptance.cpp:249-290
    kExact = 2      # exp(log g), test_fkpg.cpp:365-381
    kNegative = 3   # -0.1: ContractError, test_fkpg.cpp:436-445


class PGChains:
    def __init__(self, target: GenSSMTarget, x0, delta, root_keys: torch.Tensor, N: int,
                 trace: bool = False, pm: int = 0):
        dev = target.device
        self.target, self.N = target, int(N)
        Cn = root_keys.shape[0]
        self.C = Cn
        x0 = torch.as_tensor(x0, dtype=torch.float64, device=dev)
        if x0.dim() == 2:
            x0 = x0.unsqueeze(0).expand(Cn, -1, -1)
        T1 = target.T + 1
        self.x = x0.contiguous().clone()
        self.keys = torch.zeros((Cn, T1), dtype=torch.int64, device=dev)
        self.delta = torch.full((Cn,), float(delta), dtype=torch.float64, device=dev)
        self.iter = torch.zeros(Cn, dtype=torch.int64, device=dev)
        self.updates = torch.zeros(Cn, dtype=torch.int64, device=dev)
        self.last_update = torch.zeros(Cn, dtype=torch.float64, device=dev)
        self.root_keys = root_keys.contiguous()
        self.status = torch.zeros(Cn, dtype=torch.int32, device=dev)
        self.bad_t = torch.zeros(Cn, dtype=torch.int32, device=dev)
        self.ancestors = torch.zeros((Cn, T1, N), dtype=torch.int32, device=dev) if trace else None
        self.selected = torch.zeros((Cn, T1), dtype=torch.int32, device=dev) if trace else None
        self._ws = None
        self._ws_variant = None
        self.pm = int(pm)  # PseudoMarginal.* (fkpg.cpp:233-250 with a device estimator)

    def raw(self) -> _lib.PgChains:
        r = _lib.PgChains()
        p = lambda t: None if t is None else t.data_ptr()
        r.C, r.N = self.C, self.N
        r.x, r.keys, r.delta, r.iter = p(self.x), p(self.keys), p(self.delta), p(self.iter)
        r.updates, r.last_update, r.root_keys = p(self.updates), p(self.last_update), p(self.root_keys)
        r.status, r.bad_t = p(self.status), p(self.bad_t)
        r.ancestors, r.selected = p(self.ancestors), p(self.selected)
        r.pm_kind = self.pm
        return r

    def aux_pgibbs_step(self, variant=Variant.kReference, mode=ProposalMode.kGradient, stream=None):
        lib = _lib.load()
        tr, ch = self.target.raw(), self.raw()
        if self._ws_variant != variant:
            n = lib.auxmc_aux_pgibbs_workspace(C.byref(tr), self.C, self.N, int(variant))
            self._ws = torch.empty(n, dtype=torch.uint8, device=self.target.device)
            self._ws_variant = variant
        _lib.check(lib.auxmc_aux_pgibbs_step(
            C.byref(tr), C.byref(ch), int(mode), int(variant), self._ws.data_ptr(),
            self._ws.numel(), stream if stream is not None else torch.cuda.current_stream().cuda_stream),
            "aux_pgibbs_step")

    def adapt_delta(self, target_rate):
        ch = self.raw()
        _lib.check(_lib.load().auxmc_pg_adapt_delta(C.byref(ch), float(target_rate),
                                                    torch.cuda.current_stream().cuda_stream),
                   "pg_adapt_delta")


def init_pg(target: GenSSMTarget, x0, delta, seed: int, n_chains: int, N: int, first: int = 0,
            trace=False) -> PGChains:
    """fkpg::init_pg (fkpg.cpp:252-258) for chains rooted at from_seed(seed).derive(kChain, c)."""
    return PGChains(target, x0, delta, chain_keys(seed, n_chains, first, target.device), N, trace)
