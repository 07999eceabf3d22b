#!/usr/bin/env python
"""bench.py — device-timed throughput of the auxmc hot path on B200.

Default workload (BASELINE.json configs[1], "C2"): LGSSM pathwise posterior
sampling with the parallel-in-time prefix-sum sampler (pit::prefix_sample),
state dim 4, T = 2^16, 1024 chains per GPU sharing one Kalman filter result
(weak scaling: chains are independent; no data-path collective).  A step is
one sweep that draws every chain's full path (1024 x 65537 x 4 doubles).
Inputs (filter result, pre-drawn variates, 2.1 GB) and outputs (2.1 GB) are
far larger than the 126 MB L2, so no explicit flush is needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config c2|c1|c3|c4|c5|c5ts] [--sampler prefix|dnc|seq] [--noise predrawn|rng]

Under torchrun each rank runs its own chains; the step time is the max over
ranks (CUDA events, barrier + synchronize on both sides).  Rank 0 prints one
JSON line.  `--impl reference` times the reference algorithm on the host
cores instead (the oracle port of the reference algorithm) on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys
import threading
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "chain-timesteps/sec (device-timed) at 1/2/4/8 B200; MCMC iters/sec; % HBM/FP64 roofline"
UNIT = "chain-timesteps/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--config", default="c2", choices=["c2", "c1", "c3", "c4", "c5", "c5ts"])
    p.add_argument("--sampler", default="prefix", choices=["prefix", "dnc", "seq"])
    p.add_argument("--noise", default="predrawn", choices=["predrawn", "rng"])
    p.add_argument("--chains", type=int, default=0, help="chains per GPU (0 = config default)")
    p.add_argument("--T", type=int, default=0, help="horizon (0 = config default)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-graph", action="store_true", help="c1: eager launches, no CUDA graph")
    return p.parse_args()


def dist_env():
    from paper_2303_00301_b200.shard import dist_env as env
    return env()


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for n, v in zip(names, s[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.samples)}


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "_fallback": True}


def ncu_traffic(kernel):
    """dram read+write bytes per launch from a committed ncu --set full capture."""
    try:
        t = json.loads((ROOT / "profiles" / "traffic.json").read_text())
        return t.get(kernel)
    except Exception:
        return None


# ---------------------------------------------------------------------------- C2
def c2_setup(args, rank, device):
    import torch
    from paper_2303_00301_b200 import bench_models as bm, lgssm, rng, shard
    T = args.T or 65536
    C = args.chains or 1024
    spec = bm.ModelSpec(kind="lgssm-synthetic", T=T, dx=4, dy=1, data_seed=1)
    lat, data = bm.simulate(spec)
    model = bm.synthetic_lgssm(spec, device=device)
    fr = lgssm.kalman_filter(model, data)
    sh = shard.weak_shard(rank, int(os.environ.get("WORLD_SIZE", "1")), C)
    keys = rng.chain_keys(1, sh.count, first=sh.first, device=device)  # derive(kChain, c)
    if args.noise == "predrawn":
        term = rng.normals(keys, rng.kTerminalDraw, 0, 1, 4).reshape(C, 4)
        back = rng.normals(keys, rng.kBackwardNoise, 0, T, 4)
        noise = lgssm.Noise.predrawn(term, back, device=device)
    else:
        noise = lgssm.Noise.stream(keys)
    sampler = {"seq": 0, "prefix": 1, "dnc": 2}[args.sampler]
    if sampler == 2 and args.noise == "predrawn":
        from paper_2303_00301_b200 import pit
        nb = pit.dnc_bridge_count(T)
        noise.bridge = rng.normals(keys, rng.kDncBridge, 0, nb, 4)
    ps = lgssm.PathSampler(model, C, sampler, True)
    out = torch.empty((C, T + 1, 4), dtype=torch.float64, device=device)
    torch.cuda.synchronize()
    return dict(T=T, C=C, d=4, model=model, fr=fr, noise=noise, ps=ps, out=out, data=data,
                sampler=sampler, spec=spec)


def c2_e2e(args, st, steps, warmup, world):
    """Same sweep through the public Python API from pinned HOST buffers
    (lgssm.HostPipeline): per step the filter result and every chain's variates go
    host-to-device and every path comes back device-to-host, chunked over three
    streams so both PCIe directions and the kernels overlap."""
    import torch
    from paper_2303_00301_b200 import lgssm
    fr, noise = st["fr"], st["noise"]
    pin = lambda t: None if t is None else t.cpu().pin_memory()  # noqa: E731
    h_fr = lgssm.FilterResult(pin(fr.pred_mean), pin(fr.pred_cov), pin(fr.filt_mean),
                              pin(fr.filt_cov), pin(fr.log_marginal), fr.status.cpu())
    h_noise = lgssm.Noise(keys=pin(noise.keys), terminal=pin(noise.terminal),
                          backward=pin(noise.backward), bridge=pin(noise.bridge))
    h_out = torch.empty(st["out"].shape, dtype=torch.float64).pin_memory()
    C = st["C"]
    chunks = int(os.environ.get("AUXMC_E2E_CHUNKS", "32"))
    chunks = chunks if C % chunks == 0 else 1
    pipe = lgssm.HostPipeline(st["model"], C, st["sampler"], chunks)
    h2d = sum(t.numel() * t.element_size() for t in (h_fr.pred_mean, h_fr.pred_cov,
                                                      h_fr.filt_mean, h_fr.filt_cov,
                                                      h_fr.log_marginal)) + \
        sum(t.numel() * t.element_size() for t in (h_noise.keys, h_noise.terminal,
                                                    h_noise.backward, h_noise.bridge)
            if t is not None)
    d2h = h_out.numel() * h_out.element_size()

    def step():
        pipe(h_fr, h_noise, h_out)

    for _ in range(warmup):
        step()
    ms = timed(step, steps, world)
    ct = st["C"] * (st["T"] + 1) * steps * world
    return {"value": ct / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": ms / steps,
            "pipeline": f"{chunks} chain chunks, 3 streams (H2D | draw | D2H)"}


def timed(fn, steps, world):
    """K steps bracketed by barrier + synchronize; CUDA events; max over ranks (ms)."""
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        from paper_2303_00301_b200.shard import max_over_ranks
        ms = max_over_ranks(ms, world, device="cuda")
        dist.barrier()
    return ms


def cpu_reference_prefix(T, d, n_chains, threads, sampler="prefix", seed=1):
    """Time the CPU reference algorithm (the oracle port: the reference itself
    cannot be compiled here, Eigen3 is absent) on n_chains chains of the C2
    workload; returns (ct/s, seconds, kind)."""
    import concurrent.futures as cf
    from oracle import pyoracle as O
    kind = "port"
    s = O.spec("lgssm-synthetic", T=T, dx=d, dy=1, data_seed=1)
    lat, data = O.simulate(s)
    m = O.synthetic_lgssm(s)
    fr = O.kalman_filter(m, data)
    fn = {"prefix": O.prefix_sample, "seq": O.backward_sample, "dnc": O.dnc_sample}[sampler]

    def one(c):
        return fn(m, fr, O.stream_noise(O.derive(O.from_seed(seed), O.L_CHAIN, c)))

    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(one, range(n_chains)))
    dt = time.perf_counter() - t0
    return n_chains * (T + 1) / dt, dt, kind


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU path on this box's host cores."""
    if rank != 0:
        return
    T = args.T or 65536
    threads = os.cpu_count() or 1
    # calibrate: one chain single-threaded, then size each step to ~2 s of wall time
    v1, t1, kind = cpu_reference_prefix(T, 4, 1, 1, args.sampler)
    per_step = max(threads, int(threads * max(1.0, 2.0 / max(t1, 1e-3))))
    for _ in range(max(args.warmup, 0) and 1):
        cpu_reference_prefix(T, 4, threads, threads, args.sampler)
    vals, secs = [], 0.0
    for _ in range(args.steps):
        v, dt, kind = cpu_reference_prefix(T, 4, per_step, threads, args.sampler)
        vals.append(v)
        secs += dt
    value = per_step * (T + 1) * args.steps / secs
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": f"C2 lgssm-synthetic d=4 T={T}, pit::{args.sampler}_sample per "
                               f"chain on host cores", "chains_per_step": per_step},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"{per_step} chains x (T+1)={T + 1} per step, "
                                   f"{threads} threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_c2(args, rank, world, local):
    import torch
    from paper_2303_00301_b200 import _lib
    device = f"cuda:{local}"
    torch.cuda.set_device(local)
    lib = _lib.load()
    if lib.auxmc_device_ok() != 1:
        raise SystemExit("libauxmc_b200: no usable sm_100 device")
    st = c2_setup(args, rank, device)
    ps, fr, noise, out = st["ps"], st["fr"], st["noise"], st["out"]

    def step():
        ps(fr, noise, out)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    hot = {1: "k_prefix", 2: "k_dnc_", 0: "k_seq_sample"}[st["sampler"]]
    launches0 = lib.auxmc_launch_count()
    lib.auxmc_profile_begin()
    with Clocks(local) as clk:
        ms = timed(step, args.steps, world)
    tot = __import__("ctypes").c_double(0.0)
    cnt = __import__("ctypes").c_longlong(0)
    lib.auxmc_profile_end(hot.encode(), __import__("ctypes").byref(tot),
                          __import__("ctypes").byref(cnt))
    launches = lib.auxmc_launch_count() - launches0
    if int(ps.status.max()) != 0:
        raise SystemExit(f"sampler status {int(ps.status.max())}")
    T, C, d = st["T"], st["C"], st["d"]
    ct = C * (T + 1) * args.steps * world
    value = ct / (ms / 1e3)
    pk = peaks()
    bytes_per_ct = (16 * d if args.noise == "predrawn" else 8 * d) if st["sampler"] == 1 else \
        (32 * d if st["sampler"] == 2 else 16 * d)
    # the hot kernel's device time per step (DnC: all level launches of a sweep)
    kernel_ms = tot.value / max(args.steps, 1)
    step_bytes = bytes_per_ct * C * (T + 1)
    achieved = step_bytes / (kernel_ms / 1e3) / 1e9 if cnt.value else None
    roof = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": (achieved / pk["hbm_gbs"]) if achieved else None,
            "traffic": ncu_traffic(f"{hot}:{args.noise}:{T}:{C}"),
            "kernel": hot, "kernel_ms": kernel_ms,
            "kernel_launches_per_step": cnt.value / max(args.steps, 1), "kernel_share_of_step":
                (tot.value / ms) if ms else None,
            "algorithmic_bytes_per_chain_timestep": bytes_per_ct,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs" + (" (fallback)" if pk.get("_fallback") else "")}
    e2e = None
    if not args.no_e2e:
        e2e = c2_e2e(args, st, max(2, min(args.steps, 5)), 1, world)
    cpu = None
    if rank == 0 and not args.no_cpu:
        n = 2 if T >= 32768 else 8
        v, dt, kind = cpu_reference_prefix(T, d, n, 1, args.sampler)
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": kind,
               "sample": f"{n} chains x (T+1)={T + 1}, pit::{args.sampler}_sample, 1 thread, "
                         f"{dt:.1f} s"}
    if rank == 0:
        sampler_name = {0: "seq", 1: "prefix", 2: "dnc"}[st["sampler"]]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"C2: lgssm-synthetic d=4 dy=1 T={T}, {C} chains/GPU, "
                                   f"pit::{sampler_name}_sample from one shared Kalman filter",
                       "noise": args.noise, "chains_per_gpu": C, "T": T,
                       "parallelism": f"chains sharded over {world} GPU(s)",
                       "l2": "inputs+outputs (4.3 GB) >> L2 (126 MB); no flush needed",
                       "mcmc_sweeps_per_sec": 1e3 * args.steps / ms},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    try:
        if args.config == "c2":
            run_c2(args, rank, world, local)
        else:
            from tools import bench_aux
            bench_aux.run(args, rank, world, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
