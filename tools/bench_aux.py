"""MCMC bench configurations for bench.py (one record each; bench.py embeds them in the
headline line's `configs` or prints one as its own line with --config).

c1: auxiliary Kalman sampler, 1-D LGSSM, T = 1024, 1 chain, prefix backend with the
    scan filter (BASELINE.json configs[0]); one CUDA graph per iteration.
c3: Lorenz-96 d = 40 diffusion smoothing, auxiliary Kalman sampler, T = 4096,
    256 chains, sequential backend and filter (configs[2]).
c4: stochastic volatility d = 3, auxiliary particle Gibbs, N = 256, T = 2^14
    (configs[3]) over 148 chains (one per SM) — c4_1chain: the same for ONE chain,
    the latency case SURVEY.md §8(d) asks to report beside the full-GPU batch.
c5: spatio-temporal grid 4 (d = 16), T = 2^20, 1 chain, aux-Kalman with the scan
    filter and prefix sampler (configs[4]; one GPU per chain).
c5ts: the same iteration time-sharded over the ranks (strong scaling).

A step is one MCMC iteration of every chain on the GPU; value = chains * (T+1) *
iterations / device seconds (max over ranks).  Each record also carries the
reference's own CPU implementation (tools/cpu_ref.py, oracle/_ref) on a bounded
sample of the same workload and an e2e leg whose chain states live in pinned host
memory (H2D before and D2H after every iteration, inside the timed region).
"""
from __future__ import annotations

import ctypes

UNIT = "chain-timesteps/s"
C5_DELTA = 5e-4
# measured: DMMA m8n8k4 FP64 throughput, tools/micro/lat.cu (profiles/r1_micro_latency_fp64.txt)
FP64_PEAK_TFLOPS = 37.1
FP64_SOURCE = "measured DMMA FP64 throughput, profiles/r1_micro_latency_fp64.txt " \
              "(MEASURED_PEAKS.json carries HBM and bf16 only)"


def _cfg(name, args):
    from paper_2303_00301_b200 import auxk, bench_models as bm
    if name == "c1":
        T = args.T if args.config == "c1" and args.T else 1024
        return dict(T=T, C=1, d=1, spec=bm.ModelSpec(kind="lgssm-synthetic", T=T, dx=1, dy=1,
                                                   data_seed=1),
                    backend=auxk.Backend.kPrefix, pf=True, delta=1.0, flops=130.0,
                    bound="latency", x0="m0",
                    workload="C1 aux-Kalman 1-D LGSSM, prefix backend + scan filter, 1 chain "
                             "(one CUDA graph per iteration)")
    if name == "c3":
        T = args.T if args.config == "c3" and args.T else 4096
        C = args.chains if args.config == "c3" and args.chains else 256
        return dict(T=T, C=C, d=40, spec=bm.ModelSpec(kind="lorenz96", T=T, dx=40, data_seed=3),
                    backend=auxk.Backend.kSequential, pf=False, delta=0.05, flops=2.14e6,
                    bound="fp64", x0="latent",
                    workload="C3 aux-Kalman Lorenz-96 d=40 (q=20 exact rows), sequential "
                             "backend and filter")
    if name == "c5":
        T = args.T if args.config == "c5" and args.T else (1 << 20)
        return dict(T=T, C=1, d=16, spec=bm.ModelSpec(kind="spatio-temporal", T=T, grid=4,
                                                    data_seed=7),
                    backend=auxk.Backend.kPrefix, pf=True, delta=C5_DELTA, flops=464e3,
                    bound="fp64", x0="latent",
                    workload="C5 spatio-temporal grid 4 (d=16) aux-Kalman, scan filter + "
                             "prefix sampler, 1 chain (1 GPU: no time sharding)")
    if name in ("c4", "c4_1chain"):
        T = args.T if args.config == "c4" and args.T else 16384
        C = 1 if name == "c4_1chain" else (args.chains if args.config == "c4" and args.chains
                                             else 148)
        N, d = 256, 3
        # per (i, j) pair after whitening: d differences + d squares/FMAs + 2 scale/adds
        # + exp (20 flops) + accumulate: the minimal structure-aware count
        return dict(T=T, C=C, d=d, N=N, spec=bm.ModelSpec(kind="stochvol", T=T, dx=3,
                                                        data_seed=11),
                    delta=1.0, flops=N * N * (2 * d + 3 + 20.0), bound="fp64", x0="latent",
                    workload=f"C4 stochvol aux particle Gibbs N=256, "
                             f"{'PIT' if args.variant == 'pit' else 'reference'} cSMC, {C} chain(s)")
    raise ValueError(name)


def record(name, args, rank, world, local):
    if name == "c5ts":
        return record_c5ts(args, rank, world, local)
    import numpy as np
    import torch
    from bench import Clocks, steps_for, timed
    from paper_2303_00301_b200 import _lib, auxk, bench_models as bm, fkpg, shard
    device = f"cuda:{local}"
    lib = _lib.load()
    c = _cfg(name, args)
    T, C, d, spec = c["T"], c["C"], c["d"], c["spec"]
    lat, data = bm.simulate(spec)
    tg = auxk.make_target(spec, data, device=device)
    x0 = torch.as_tensor(lat, device=device) if c["x0"] == "latent" else \
        torch.as_tensor(lat * 0 + tg.m0.cpu().numpy(), device=device)
    sh = shard.weak_shard(rank, world, C)
    pg = name.startswith("c4")
    if pg:
        variant = fkpg.Variant.kPit if args.variant == "pit" else fkpg.Variant.kReference
        ch = fkpg.init_pg(tg, x0, c["delta"], 1, sh.count, c["N"], first=sh.first)

        def step():
            ch.aux_pgibbs_step(variant)
    else:
        ch = auxk.init_chains(tg, x0, c["delta"], 1, sh.count, first=sh.first)
        use_graph = name == "c1" and not args.no_graph

        def step():
            if use_graph:
                ch.graph_step(c["backend"], parallel_filter=c["pf"])
            else:
                ch.kernel_step(c["backend"], parallel_filter=c["pf"])

    warm = max(args.warmup, 1) if name != "c3" else 1
    for _ in range(warm):
        step()
    torch.cuda.synchronize()
    one = timed(step, 1, world)
    steps = steps_for(one, args.min_time, 1)
    n0 = lib.auxmc_launch_count()
    with Clocks(local) as clk:
        ms = timed(step, steps, world)
    launches = lib.auxmc_launch_count() - n0
    if not pg and getattr(ch, "graph_launches", None) and launches == 0:
        launches = ch.graph_launches(c["backend"], parallel_filter=c["pf"]) * steps
    ct = C * (T + 1) * steps * world
    value = ct / (ms / 1e3)
    tflops = c["flops"] * ct / (ms / 1e3) / 1e12
    cfg = {"workload": c["workload"], "T": T, "chains_per_gpu": C,
           "mcmc_iters_per_sec": 1e3 * steps / ms,
           "l2": "chain states and per-step elements exceed L2 (126 MB) except c1/c4_1chain, "
                 "whose working set is L2-resident by design (latency-bound)"}
    if pg:
        st_bad = int(ch.status.max())
        cfg["update_rate"] = float(ch.updates.sum()) / max(1, float(ch.iter.sum()))
        cfg["status_max"] = st_bad
        if name == "c4":
            cfg["N"] = c["N"]
    else:
        cfg["accept_rate"] = float(ch.accepted.sum()) / max(1, float(
            (ch.accepted + ch.rejected).sum()))
        cfg["aborted"] = int(ch.aborted.sum())
        cfg["delta"] = c["delta"]
    rec = {"value": value, "unit": UNIT, "ms_per_step": ms / steps, "steps": steps,
           "warmup": warm, "config": cfg,
           "roofline": {"bound": c["bound"], "achieved": tflops, "peak": FP64_PEAK_TFLOPS,
                        "unit": "TFLOP/s", "frac": tflops / FP64_PEAK_TFLOPS, "traffic": None,
                        "algorithmic_flops_per_chain_timestep": c["flops"],
                        "peak_source": FP64_SOURCE},
           "gpu_launches": int(launches), "clocks": clk.summary()}
    if not args.no_e2e:
        rec["e2e"] = e2e_host_states(ch, step, pg, max(1, min(steps, 5)), world, C, T)
    if rank == 0 and world == 1 and not args.no_cpu:
        rec["cpu_baseline"] = cpu_record(name, c)
    return rec


def e2e_host_states(ch, step, pg, steps, world, C, T):
    """Chain states resident in pinned HOST memory: every iteration copies the paths
    (and particle-Gibbs keys) host-to-device, runs the step, and copies paths, keys and
    the accept/update statistics back, inside the timed region."""
    import torch
    from bench import timed
    h_x = torch.empty(ch.x.shape, dtype=ch.x.dtype).pin_memory()
    h_x.copy_(ch.x)
    extra_in = [(ch.keys, torch.empty(ch.keys.shape, dtype=ch.keys.dtype).pin_memory())] if pg else []
    outs = [(ch.updates, ch.last_update, ch.status)] if pg else [(ch.stats,)]
    h_out = [torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in outs[0]]
    for dev, host in extra_in:
        host.copy_(dev)

    def e2e_step():
        ch.x.copy_(h_x, non_blocking=True)
        for dev, host in extra_in:
            dev.copy_(host, non_blocking=True)
        step()
        h_x.copy_(ch.x, non_blocking=True)
        for dev, host in extra_in:
            host.copy_(dev, non_blocking=True)
        for dev, host in zip(outs[0], h_out):
            host.copy_(dev, non_blocking=True)

    e2e_step()
    ms = timed(e2e_step, steps, world)
    nb_x = h_x.numel() * h_x.element_size()
    nb_in = nb_x + sum(h.numel() * h.element_size() for _, h in extra_in)
    nb_out = nb_in + sum(h.numel() * h.element_size() for h in h_out)
    return {"value": C * (T + 1) * steps * world / (ms / 1e3), "unit": UNIT,
            "h2d_bytes_per_step": nb_in, "d2h_bytes_per_step": nb_out, "ms_per_step": ms / steps,
            "steps": steps, "pipeline": "chain states in pinned host memory; H2D, iteration, "
                                        "D2H on one stream"}


def cpu_record(name, c):
    """The reference's CPU implementation (oracle/_ref) on a bounded sample of the same
    workload; per chain-timestep cost is linear in T (acceptance.cpp criterion 1:
    slope 0.968, profiles/r2_ref/acceptance.txt), so reduced-T samples are stated."""
    from oracle import pyoracle as O
    from tools import cpu_ref as CR
    P = CR.host_cores()
    if name == "c1":
        s = O.spec("lgssm-synthetic", T=c["T"], dx=1, dy=1, data_seed=1)
        one = CR.aux_baseline(s, 60, 1, 1, 1, True, 1.0, label="1 core: ")
        allw = CR.aux_baseline(s, 20, 1, 1, 1, True, 1.0, workers=P, label="workers=nproc: ")
        one["workers_nproc"] = {k: allw[k] for k in ("value", "cores", "sample")}
        return one
    if name == "c3":  # the full horizon: one kernel_step per host thread (~10 s)
        s = O.spec("lorenz96", T=c["T"], dx=40, data_seed=3)
        return CR.aux_baseline(s, 1, P, P, 0, False, 0.05, label="full T: ")
    if name == "c5":
        s = O.spec("spatio-temporal", T=16384, grid=4, data_seed=7)
        one = CR.aux_baseline(s, 1, 1, 1, 1, True, C5_DELTA, label="reduced T, 1 core: ")
        allw = CR.aux_baseline(s, 1, 1, 1, 1, True, C5_DELTA, workers=P,
                               label="reduced T, workers=nproc: ")
        one["workers_nproc"] = {k: allw[k] for k in ("value", "cores", "sample")}
        return one
    if name == "c4":
        s = O.spec("stochvol", T=4096, dx=3, data_seed=11)
        return CR.pg_baseline(s, 256, 1, P, P, label="reduced T, reference sequential cSMC: ")
    if name == "c4_1chain":
        s = O.spec("stochvol", T=4096, dx=3, data_seed=11)
        return CR.pg_baseline(s, 256, 1, 1, 1, label="reduced T, 1 chain, 1 core: ")
    return None


def record_c5ts(args, rank, world, local):
    """C5 time-sharded: the full auxiliary Kalman iteration of ONE chain on the C5 target
    (spatio-temporal grid 4, d = 16, T = 2^20) with the horizon split over the ranks
    (tshard.ShardedAuxChain); strong scaling (T fixed).  A step = one MCMC iteration
    including the exchanges."""
    import torch
    from bench import Clocks, steps_for, timed
    from paper_2303_00301_b200 import _lib, auxk, bench_models as bm, tshard
    device = f"cuda:{local}"
    T = args.T or (1 << 20)
    spec = bm.ModelSpec(kind="spatio-temporal", T=T, grid=4, data_seed=7)
    lat, data = bm.simulate(spec)
    tg = auxk.make_target(spec, data, device=device)
    ch = auxk.init_chains(tg, torch.as_tensor(lat, device=device), C5_DELTA, 1, 1)
    if world > 1:
        exchange = tshard.torch_exchange()
    else:
        def exchange(t):
            return [t]
    lib = _lib.load()
    sa = tshard.ShardedAuxChain(ch, rank, world, exchange)

    def step():
        sa.step()

    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize()
    steps = steps_for(timed(step, 1, world), args.min_time, args.steps)
    n0 = lib.auxmc_launch_count()
    with Clocks(local) as clk:
        ms = timed(step, steps, world)
    launches = lib.auxmc_launch_count() - n0
    value = (T + 1) * steps / (ms / 1e3)
    F_pit = 464e3
    tflops = F_pit * value / 1e12
    g = tshard.TShardGeom.of(T, 16)
    return {"value": value, "unit": UNIT, "ms_per_step": ms / steps, "steps": steps,
            "warmup": max(args.warmup, 1),
            "config": {"workload": "C5 spatio-temporal grid 4 (d=16) aux-Kalman iteration, "
                                   "1 chain, time-sharded (forward/reverse scan filter + "
                                   "prefix sampler split over ranks)", "T": T,
                       "accept_rate": float(ch.accepted.sum()) / max(1, float(
                           (ch.accepted + ch.rejected).sum())),
                       "super_blocks": g.nsup, "super_block_steps": g.SB,
                       "parallelism": f"time sharded over {world} GPU(s)"},
            "roofline": {"bound": "fp64", "achieved": tflops, "peak": FP64_PEAK_TFLOPS,
                         "unit": "TFLOP/s", "frac": tflops / FP64_PEAK_TFLOPS, "traffic": None,
                         "algorithmic_flops_per_chain_timestep": F_pit, "peak_source": FP64_SOURCE},
            "gpu_launches": int(launches), "clocks": clk.summary()}
