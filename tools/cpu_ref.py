"""CPU legs of bench.py: the REFERENCE's own implementation timed on this box's host
cores (oracle/_ref — /root/reference/proj/src compiled unmodified against the shims,
driven through oracle/refbridge.py), with the C restatement (oracle/pyoracle.py) as
the fallback when _ref is missing.  Test/measurement infrastructure: never on the
product path.  ctypes releases the GIL during a call, so a thread pool over chains
runs the reference's re-entrant API on every core (SURVEY.md §8(b) threading note).

Every function returns a dict {value (chain-timesteps/s), seconds, kind, cores,
sample} for a bounded sample of the named workload.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import time

import numpy as np

from oracle import pyoracle as O

try:
    from oracle import refbridge as R
except Exception:  # pragma: no cover
    R = None


def have_ref() -> bool:
    return R is not None and R.available()


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _pool(fn, items, threads):
    if threads <= 1:
        return [fn(i) for i in items]
    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        return list(ex.map(fn, items))


# ---------------------------------------------------------------- C2: pathwise draws
class C2Ref:
    """pit::prefix_sample / dnc_sample / lgssm::backward_sample per chain from one shared
    Kalman filter result (models.cpp:338-344 model), pre-drawn variates read through a
    NoiseSource (rng.hpp:123-126) or StreamNoise (on-the-fly Box-Muller)."""

    def __init__(self, T, d=4, sampler="prefix", noise="predrawn", n_noise=1):
        self.T, self.d, self.sampler, self.noise = T, d, sampler, noise
        s = O.spec("lgssm-synthetic", T=T, dx=d, dy=1, data_seed=1)
        _, data = O.simulate(s)
        self.m = O.synthetic_lgssm(s)
        self.kind = "reference" if have_ref() else "port"
        if self.kind == "reference":
            self.rm = R.RModel(self.m)
            self.fr = R.kalman_filter(self.rm, data)
            self.fn = {"prefix": R.prefix_sample, "seq": R.backward_sample,
                       "dnc": R.dnc_sample}[sampler]
        else:
            self.fr = O.kalman_filter(self.m, data)
            self.fn = {"prefix": O.prefix_sample, "seq": O.backward_sample,
                       "dnc": O.dnc_sample}[sampler]
        rng = np.random.default_rng(7)
        nb = 2 * T + 2
        # a few variate sets, reused round-robin (the work does not depend on the values)
        self.pre = [dict(terminal=rng.standard_normal(d), backward=rng.standard_normal((T, d)),
                         bridge=rng.standard_normal((nb, d)) if sampler == "dnc" else None)
                    for _ in range(n_noise)]

    def one(self, c):
        if self.noise == "rng":
            root = O.derive(O.from_seed(1), O.L_CHAIN, c)
            if self.kind == "reference":
                return self.fn(self.rm, self.fr, root)
            return self.fn(self.m, self.fr, O.stream_noise(root))
        p = self.pre[c % len(self.pre)]
        if self.kind == "reference":
            return self.fn(self.rm, self.fr, p)
        nz, keep = O.predrawn_noise(self.d, p["terminal"], p["backward"], p["bridge"])
        return self.fn(self.m, self.fr, nz)

    def run(self, chains, threads):
        t0 = time.perf_counter()
        _pool(self.one, range(chains), threads)
        dt = time.perf_counter() - t0
        return chains * (self.T + 1) / dt, dt


def c2_baseline(T, sampler, noise, threads, target_s=3.0):
    ref = C2Ref(T, 4, sampler, noise, n_noise=min(threads, 4))
    _, t1 = ref.run(1, 1)  # calibrate (and warm up)
    per_thread = max(1, int(round(target_s / max(t1, 1e-3))))
    chains = per_thread * threads
    v, dt = ref.run(chains, threads)
    return {"value": v, "unit": "chain-timesteps/s", "cores": threads, "kind": ref.kind,
            "seconds": dt,
            "sample": f"{chains} chains x (T+1)={T + 1}, pit::{sampler}_sample "
                      f"({noise} variates), one shared filter, {threads} threads, {dt:.1f} s"}


# ---------------------------------------------------------------- aux Kalman chains
def _target(spec, data):
    if have_ref():
        return R.make_target(spec, data), "reference"
    return O.make_target(spec, data), "port"


def aux_baseline(spec, iters, chains, threads, backend, parallel, delta, workers=1, x0=None,
                 label=""):
    """kernel_step (auxk.cpp:130-198) for `chains` independent chains x `iters` iterations,
    chains spread over `threads` host threads; workers = the reference's intra-chain
    thread count (KernelOptions::workers)."""
    lat, data = O.simulate(spec)
    tg, kind = _target(spec, data)
    if x0 is None:
        x0 = np.repeat(O.make_target(spec, data).arrays()["m0"][None, :], spec.T + 1, 0)
    Chain = R.AuxChain if kind == "reference" else O.AuxChain

    def one(c):
        ch = Chain(tg, x0, delta)
        root = O.derive(O.from_seed(1), O.L_CHAIN, c)
        for _ in range(iters):
            if kind == "reference":
                ch.step(root, backend, parallel, 0, workers)
            else:
                ch.step(root, backend, int(parallel), 0)
        return ch

    t0 = time.perf_counter()
    _pool(one, range(chains), threads)
    dt = time.perf_counter() - t0
    T = spec.T
    v = chains * (T + 1) * iters / dt
    return {"value": v, "unit": "chain-timesteps/s", "cores": max(threads, workers), "kind": kind,
            "seconds": dt, "iters_per_sec_per_chain": iters / dt * (threads / max(chains, 1)),
            "sample": f"{label}{chains} chain(s) x {iters} kernel_step(s) at T={T}, "
                      f"{threads} thread(s){', workers=' + str(workers) if workers > 1 else ''}, "
                      f"{dt:.1f} s"}


def pg_baseline(spec, N, iters, chains, threads, delta=1.0, mode=1, label=""):
    """aux_pgibbs_step (fkpg.cpp:252-271), the reference's sequential cSMC."""
    lat, data = O.simulate(spec)
    tg, kind = _target(spec, data)
    x0 = np.tile(np.full(O.latent_dim(spec), spec.sv_mu), (spec.T + 1, 1))
    Chain = R.PGChain if kind == "reference" else O.PGChain

    def one(c):
        ch = Chain(tg, x0, delta)
        root = O.derive(O.from_seed(1), O.L_CHAIN, c)
        for _ in range(iters):
            ch.step(N, root, mode=mode)
        return ch

    t0 = time.perf_counter()
    _pool(one, range(chains), threads)
    dt = time.perf_counter() - t0
    v = chains * (spec.T + 1) * iters / dt
    return {"value": v, "unit": "chain-timesteps/s", "cores": threads, "kind": kind,
            "seconds": dt,
            "sample": f"{label}{chains} chain(s) x {iters} aux_pgibbs_step(s), N={N}, T={spec.T}, "
                      f"{threads} thread(s), {dt:.1f} s"}
