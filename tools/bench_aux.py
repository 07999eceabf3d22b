"""Secondary bench configurations (bench.py --config c1|c3|c4), one JSON line each.

c1: auxiliary Kalman sampler, 1-D LGSSM, T = 1024, 1 chain, prefix backend
    (BASELINE.json configs[0]); a step is one MCMC iteration.
c3: Lorenz-96 d = 40 diffusion smoothing, auxiliary Kalman sampler, T = 4096,
    256 chains, sequential backend (configs[2]).
c4: stochastic volatility d = 3, auxiliary particle Gibbs, N = 256, T = 2^14
    (configs[3]), parallel-in-time cSMC (--sampler dnc selects the reference cSMC).
c5: spatio-temporal grid 4 (d = 16), T = 2^20, 1 chain, aux-Kalman with the scan
    filter and prefix sampler (configs[4]; one GPU per chain).
c5ts: the same iteration time-sharded over the ranks (strong scaling).
Units: chain-timesteps/s = chains * (T+1) * iterations / device seconds.
"""
from __future__ import annotations

import ctypes
import json

METRIC = "chain-timesteps/sec (device-timed) at 1/2/4/8 B200; MCMC iters/sec; % HBM/FP64 roofline"
C5_DELTA = 5e-4
FP64_PEAK_TFLOPS = 37.1  # measured: DMMA m8n8k4 throughput, tools/micro/lat.cu (profiles/r1_micro_latency_fp64.txt)


def run(args, rank, world, local):
    import torch
    from bench import Clocks, timed
    from paper_2303_00301_b200 import _lib, auxk, bench_models as bm, fkpg, shard
    device = f"cuda:{local}"
    torch.cuda.set_device(local)
    lib = _lib.load()
    cfg = args.config
    if cfg == "c1":
        T, C, d = args.T or 1024, args.chains or 1, 1
        spec = bm.ModelSpec(kind="lgssm-synthetic", T=T, dx=1, dy=1, data_seed=1)
        backend, delta = auxk.Backend.kPrefix, 1.0
        flops_ct = 130.0  # F_pit, scan filter counted
    elif cfg == "c3":
        T, C, d = args.T or 4096, args.chains or 256, 40
        spec = bm.ModelSpec(kind="lorenz96", T=T, dx=40, data_seed=3)
        backend, delta = auxk.Backend.kSequential, 0.05
        flops_ct = 2.14e6  # F_seq at d = 40, q = 20
    elif cfg == "c5ts":
        T, C, d = args.T or (1 << 20), 1, 16
        spec, backend, delta, flops_ct = None, None, None, 464e3
    elif cfg == "c5":
        T, C, d = args.T or (1 << 20), args.chains or 1, 16
        spec = bm.ModelSpec(kind="spatio-temporal", T=T, grid=4, data_seed=7)
        backend = auxk.Backend.kDnc if args.sampler == "dnc" else auxk.Backend.kPrefix
        # log α scales with d·T: δ = 5e-4 accepts about 2/3 of moves at T = 2^20
        # (δ = 0.002 → |log α| ≈ 13, δ = 0.5 → 1.8e5); the cost does not depend on δ
        delta = C5_DELTA
        flops_ct = 464e3  # F_pit at d = 16
    else:
        T, C, d = args.T or 16384, args.chains or 148, 3
        spec = bm.ModelSpec(kind="stochvol", T=T, dx=3, data_seed=11)
        delta = 1.0
        N = 256
        # per (i, j) pair after whitening (L_Q^{-1} applied once per particle, not per
        # pair): d differences + d squares/FMAs + 2 scale/adds + exp (counted as 20
        # flops) + accumulate — the minimal structure-aware count, below SURVEY's
        # N^2 (3d^2 + d + exp) which assumed a triangular solve per pair
        flops_ct = N * N * (2 * d + 3 + 20.0)
    if cfg == "c5ts":
        return run_c5ts(args, rank, world, local, device)
    lat, data = bm.simulate(spec)
    tg = auxk.make_target(spec, data, device=device)
    x0 = torch.as_tensor(lat, device=device) if cfg != "c1" else \
        torch.as_tensor(lat * 0 + tg.m0.cpu().numpy(), device=device)
    if cfg == "c4":
        variant = fkpg.Variant.kReference if args.sampler == "dnc" else fkpg.Variant.kPit
        sh = shard.weak_shard(rank, world, C)
        ch = fkpg.init_pg(tg, x0, delta, 1, sh.count, N, first=sh.first)

        def step():
            ch.aux_pgibbs_step(variant)
    else:
        sh = shard.weak_shard(rank, world, C)
        ch = auxk.init_chains(tg, x0, delta, 1, sh.count, first=sh.first)

        # C1 / C5 are single chains: the scan filter (KernelOptions::parallel_filter)
        # parallelizes the horizon; C3 has 256 chains and uses the sequential filter.
        pf = cfg in ("c1", "c5")
        # C1 is launch-bound (~36 small kernels per iteration): replay the step as
        # one CUDA graph.  The others are long kernels; eager launches.
        use_graph = cfg == "c1" and not args.no_graph

        def step():
            if use_graph:
                ch.graph_step(backend, parallel_filter=pf)
            else:
                ch.kernel_step(backend, parallel_filter=pf)

    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize()
    n0 = lib.auxmc_launch_count()
    with Clocks(local) as clk:
        ms = timed(step, args.steps, world)
    launches = lib.auxmc_launch_count() - n0
    if cfg not in ("c4",) and getattr(ch, "graph_launches", None) and \
            ch.graph_launches(backend, parallel_filter=pf) and launches == 0:
        launches = ch.graph_launches(backend, parallel_filter=pf) * args.steps  # graph replays
    ct = C * (T + 1) * args.steps * world
    value = ct / (ms / 1e3)
    tflops = flops_ct * ct / (ms / 1e3) / 1e12
    if rank == 0:
        extra = {}
        if cfg != "c4":
            extra["accept_rate"] = float(ch.accepted.sum()) / max(1, float(
                (ch.accepted + ch.rejected).sum()))
        else:
            extra["update_rate"] = float(ch.updates.sum()) / max(1, float(ch.iter.sum()))
        line = {
            "metric": METRIC, "value": value, "unit": "chain-timesteps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": {"c1": "C1 aux-Kalman 1-D LGSSM prefix backend"
                                          + (" (CUDA graph per iteration)" if cfg == "c1" and
                                             not args.no_graph else ""),
                                    "c3": "C3 aux-Kalman Lorenz-96 d=40 sequential backend",
                                    "c4": "C4 stochvol aux particle Gibbs N=256",
                                    "c5": "C5 spatio-temporal grid 4 (d=16) aux-Kalman, scan "
                                          "filter + prefix sampler, 1 chain (1 GPU: no time "
                                          "sharding)"}[cfg],
                       "T": T, "chains_per_gpu": C, "mcmc_iters_per_sec": 1e3 * args.steps / ms,
                       **extra},
            "roofline": {"bound": "fp64" if cfg != "c1" else "latency",
                         "achieved": tflops, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": tflops / FP64_PEAK_TFLOPS, "traffic": None,
                         "algorithmic_flops_per_chain_timestep": flops_ct,
                         "peak_source": "measured DMMA FP64 throughput (profiles/r1_micro_latency_fp64.txt)"},
            "cpu_baseline": None, "e2e": None, "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)


def run_c5ts(args, rank, world, local, device):
    """C5 time-sharded: the full auxiliary Kalman iteration of ONE chain on the C5
    target (spatio-temporal grid 4, d = 16, T = 2^20) with the horizon split over
    the ranks (tshard.ShardedAuxChain): forward filter, path draw and reverse filter
    time-sharded, per-t model work repeated; strong scaling (T fixed).  A step =
    one MCMC iteration including the all-gathers."""
    import torch
    from bench import Clocks, timed
    from paper_2303_00301_b200 import _lib, auxk, bench_models as bm, tshard
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
    n0 = lib.auxmc_launch_count()
    with Clocks(local) as clk:
        ms = timed(step, args.steps, world)
    launches = lib.auxmc_launch_count() - n0
    value = (T + 1) * args.steps / (ms / 1e3)
    F_pit = 464e3  # per chain-timestep at d = 16, as the c5 line
    tflops = F_pit * value / 1e12
    if rank == 0:
        g = tshard.TShardGeom.of(T, 16)
        line = {
            "metric": METRIC, "value": value, "unit": "chain-timesteps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": "C5 spatio-temporal grid 4 (d=16) aux-Kalman iteration, "
                                   "1 chain, time-sharded (forward/reverse scan filter + "
                                   "prefix sampler split over ranks)", "T": T,
                       "accept_rate": float(ch.accepted.sum()) / max(1, float(
                           (ch.accepted + ch.rejected).sum())),
                       "super_blocks": g.nsup, "super_block_steps": g.SB,
                       "parallelism": f"time sharded over {world} GPU(s), all-gather per phase"},
            "roofline": {"bound": "fp64", "achieved": tflops, "peak": FP64_PEAK_TFLOPS,
                         "unit": "TFLOP/s", "frac": tflops / FP64_PEAK_TFLOPS, "traffic": None,
                         "algorithmic_flops_per_chain_timestep": F_pit,
                         "peak_source": "measured DMMA FP64 throughput "
                                        "(profiles/r1_micro_latency_fp64.txt)"},
            "cpu_baseline": None, "e2e": None, "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
