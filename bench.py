#!/usr/bin/env python
"""bench.py — device-timed throughput of the auxmc hot path on B200.

Headline (BASELINE.json configs[1], "C2"): LGSSM pathwise posterior sampling with the
parallel-in-time prefix-sum sampler (pit::prefix_sample), state dim 4, T = 2^16,
1024 chains per GPU sharing one Kalman filter result (weak scaling: chains are
independent; no data-path collective).  A step is one sweep that draws every chain's
full path (1024 x 65537 x 4 doubles) from pre-drawn variates resident in HBM.
Inputs (filter result, variates, 2.1 GB) and outputs (2.1 GB) are far larger than
the 126 MB L2, so no flush is needed between steps.

The same JSON line carries `configs`: one record per other BASELINE config, each
device-timed over >= 1 s with its own roofline, CPU reference baseline and e2e leg —
c2_rng (C2 with on-device Box-Muller, the like-for-like partner of the reference's
StreamNoise), c1 (aux-Kalman, 1-D LGSSM, T = 1024, 1 chain), c3 (aux-Kalman,
Lorenz-96 d = 40, T = 4096, 256 chains), c4 / c4_1chain (aux particle Gibbs, stochvol,
N = 256, T = 2^14: 148 chains and 1 chain), c5 (aux-Kalman, spatio-temporal d = 16,
T = 2^20, 1 chain).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config all|c2|c1|c3|c4|c5|c5ts] [--sampler prefix|dnc|seq]
                    [--noise predrawn|rng] [--no-configs] [--no-e2e] [--no-cpu]

--gpus N > 1 without a torchrun environment re-launches itself under
torch.distributed.run with N processes; under torchrun WORLD_SIZE must equal N.
Each rank runs its own chains; step times are the max over ranks (CUDA events,
barrier + synchronize on both sides).  Rank 0 prints one JSON line.

`--impl reference` times the reference's own CPU implementation (oracle/_ref: the
unmodified /root/reference sources compiled against the Eigen shim) on all host cores
for the headline workload, on rank 0.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import pathlib
import random
import statistics
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
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--config", default="all", choices=["all", "c2", "c1", "c3", "c4", "c5", "c5ts"])
    p.add_argument("--sampler", default="prefix", choices=["prefix", "dnc", "seq"])
    p.add_argument("--noise", default="predrawn", choices=["predrawn", "rng"])
    p.add_argument("--chains", type=int, default=0, help="chains per GPU (0 = config default)")
    p.add_argument("--T", type=int, default=0, help="horizon (0 = config default)")
    p.add_argument("--variant", default="pit", choices=["pit", "reference"],
                   help="c4: cSMC variant")
    p.add_argument("--min-time", type=float, default=1.0,
                   help="sub-config timed regions last at least this many seconds")
    p.add_argument("--no-configs", action="store_true", help="headline line only")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-graph", action="store_true", help="c1: eager launches, no CUDA graph")
    p.add_argument("--no-check", action="store_true", help="skip the reference spot check")
    return p.parse_args()


def dist_env():
    from paper_2303_00301_b200.shard import dist_env as env
    return env()


def maybe_self_launch(args):
    """`--gpus N` with N > 1 outside torchrun: re-exec under torch.distributed.run."""
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
        return
    if args.gpus <= 1:
        return
    port = str(random.randint(20000, 40000))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", port, str(ROOT / "bench.py")] + sys.argv[1:]
    os.execv(sys.executable, cmd)


class Clocks:
    """SM clock and throttle reasons sampled through NVML every ~2 ms DURING the timed
    region (B200_PROFILING.md clocks line); nvidia-smi's 100 ms period would miss
    short regions."""

    BITS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
            "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index, self.samples, self.h, self.stop = index, [], None, threading.Event()

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            idx = self.index
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            if vis and all(v.strip().isdigit() for v in vis.split(",")):
                idx = int(vis.split(",")[self.index])
            self.N, self.h = N, N.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self._sample()  # one at the region's start: short regions get >= 2 samples
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
        except Exception:
            self.h = None
        return self

    def _sample(self):
        N = self.N
        try:
            self.samples.append((N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM),
                                 N.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
        except Exception:
            pass

    def _poll(self):
        while not self.stop.is_set():
            self._sample()
            time.sleep(0.002)

    def __exit__(self, *a):
        if self.h is not None:
            self._sample()  # and one at its end, before the device work drains
        self.stop.set()
        if self.h is not None:
            self.thread.join(timeout=1)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = sorted({n for _, r in self.samples for n, b in self.BITS.items() if r & b})
        return {"sm_mhz": statistics.median(s for s, _ in self.samples),
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples),
                "source": "NVML, 2 ms period"}


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


def steps_for(one_ms, min_time_s, floor):
    """Step count so a timed region lasts >= min_time_s (clocks get sampled)."""
    return max(floor, int(min_time_s * 1e3 / max(one_ms, 1e-3)) + 1)


# ---------------------------------------------------------------------------- C2
def c2_setup(args, rank, world, device, noise_mode):
    import torch
    from paper_2303_00301_b200 import bench_models as bm, lgssm, rng, shard
    T = args.T or 65536
    C = args.chains or 1024
    spec = bm.ModelSpec(kind="lgssm-synthetic", T=T, dx=4, dy=1, data_seed=1)
    lat, data = bm.simulate(spec)
    model = bm.synthetic_lgssm(spec, device=device)
    fr = lgssm.kalman_filter(model, data)
    sh = shard.weak_shard(rank, world, C)
    keys = rng.chain_keys(1, sh.count, first=sh.first, device=device)  # derive(kChain, c)
    sampler = {"seq": 0, "prefix": 1, "dnc": 2}[args.sampler]
    if noise_mode == "predrawn":
        term = rng.normals(keys, rng.kTerminalDraw, 0, 1, 4).reshape(C, 4)
        back = rng.normals(keys, rng.kBackwardNoise, 0, T, 4)
        noise = lgssm.Noise.predrawn(term, back, device=device)
        if sampler == 2:
            from paper_2303_00301_b200 import pit
            noise.bridge = rng.normals(keys, rng.kDncBridge, 0, pit.dnc_bridge_count(T), 4)
    else:
        noise = lgssm.Noise.stream(keys)
    ps = lgssm.PathSampler(model, C, sampler, True)
    out = torch.empty((C, T + 1, 4), dtype=torch.float64, device=device)
    torch.cuda.synchronize()
    return dict(T=T, C=C, d=4, model=model, fr=fr, noise=noise, ps=ps, out=out, data=data,
                sampler=sampler, spec=spec, first=sh.first, noise_mode=noise_mode)


def c2_e2e(st, steps, warmup, world):
    """The same sweep through the public Python API from pinned HOST buffers
    (lgssm.HostPipeline): per step the filter result and every chain's variates (or
    stream keys) go host-to-device and every path comes back device-to-host, chunked
    over three streams so both PCIe directions and the kernels overlap."""
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
            "d2h_bytes_per_step": d2h, "ms_per_step": ms / steps, "steps": steps,
            "pipeline": f"{chunks} chain chunks, 3 streams (H2D | draw | D2H)"}


def c2_spot_check(st, chains=(0, -1)):
    """Outside the timed region: the device paths of two chains against the reference
    itself (oracle/_ref pit::prefix_sample on the same model, filter and streams)."""
    import numpy as np
    from oracle import pyoracle as O
    from tools import cpu_ref as CR
    T, C = st["T"], st["C"]
    s = O.spec("lgssm-synthetic", T=T, dx=4, dy=1, data_seed=1)
    _, data = O.simulate(s)
    m = O.synthetic_lgssm(s)
    if CR.have_ref():
        R = CR.R
        rm = R.RModel(m)
        fr = R.kalman_filter(rm, data)
        fn = {0: R.backward_sample, 1: R.prefix_sample, 2: R.dnc_sample}[st["sampler"]]
        kind = "reference"
        draw = lambda root: fn(rm, fr, root)  # noqa: E731
    else:
        fr = O.kalman_filter(m, data)
        fn = {0: O.backward_sample, 1: O.prefix_sample, 2: O.dnc_sample}[st["sampler"]]
        kind = "port"
        draw = lambda root: fn(m, fr, O.stream_noise(root))  # noqa: E731
    worst = 0.0
    idx = []
    for c in chains:
        c = c % C
        want = draw(O.derive(O.from_seed(1), O.L_CHAIN, st["first"] + c))
        got = st["out"][c].cpu().numpy()
        worst = max(worst, float(np.max(np.abs(got - want) / np.maximum(1.0, np.abs(want)))))
        idx.append(st["first"] + c)
    return {"chains": idx, "checker": kind, "max_rel_err": worst, "tolerance": 1e-9,
            "pass": worst <= 1e-9}


def run_c2(args, rank, world, local, noise_mode, min_time=0.0, headline=True):
    import torch
    from paper_2303_00301_b200 import _lib
    device = f"cuda:{local}"
    lib = _lib.load()
    st = c2_setup(args, rank, world, device, noise_mode)
    ps, fr, noise, out = st["ps"], st["fr"], st["noise"], st["out"]

    def step():
        ps(fr, noise, out)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    steps = args.steps
    if min_time > 0:
        steps = steps_for(timed(step, 1, world), min_time, args.steps)
    hot = {1: "k_prefix", 2: "k_dnc_", 0: "k_seq_sample"}[st["sampler"]]
    launches0 = lib.auxmc_launch_count()
    lib.auxmc_profile_begin()
    with Clocks(local) as clk:
        ms = timed(step, steps, world)
    tot, cnt = ctypes.c_double(0.0), ctypes.c_longlong(0)
    lib.auxmc_profile_end(hot.encode(), ctypes.byref(tot), ctypes.byref(cnt))
    launches = lib.auxmc_launch_count() - launches0
    if int(ps.status.max()) != 0:
        raise SystemExit(f"sampler status {int(ps.status.max())}")
    T, C, d = st["T"], st["C"], st["d"]
    ct = C * (T + 1) * steps * world
    value = ct / (ms / 1e3)
    pk = peaks()
    if st["sampler"] == 1:
        bytes_per_ct = 16 * d if noise_mode == "predrawn" else 8 * d
    else:
        bytes_per_ct = 32 * d if st["sampler"] == 2 else 16 * d
    kernel_ms = tot.value / max(steps, 1)
    step_bytes = bytes_per_ct * C * (T + 1)
    achieved = step_bytes / (kernel_ms / 1e3) / 1e9 if cnt.value else None
    if noise_mode == "predrawn":
        roof = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": (achieved / pk["hbm_gbs"]) if achieved else None,
                "traffic": ncu_traffic(f"{hot}:{noise_mode}:{T}:{C}"),
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" + (" (fallback)" if pk.get("_fallback") else "")}
    else:
        # device Box-Muller: per chain-timestep d normals = d (log + cos + sqrt) plus the
        # integer mixing; bound by the FP64 transcendental pipe, HBM traffic is 8d B
        roof = {"bound": "fp64-transcendental", "achieved_hbm_gbs": achieved,
                "peak_hbm_gbs": pk["hbm_gbs"], "hbm_frac": (achieved / pk["hbm_gbs"]) if achieved else None,
                "normals_per_sec": 4 * ct / (ms / 1e3),
                "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    roof.update({"kernel": hot, "kernel_ms": kernel_ms,
                 "kernel_launches_per_step": cnt.value / max(steps, 1),
                 "kernel_share_of_step": (tot.value / ms) if ms else None,
                 "algorithmic_bytes_per_chain_timestep": bytes_per_ct})
    check = None
    if rank == 0 and not args.no_check and headline:
        check = c2_spot_check(st)
        if not check["pass"]:
            raise SystemExit(f"spot check against the reference failed: {check}")
    e2e = None
    if not args.no_e2e:
        e2e = c2_e2e(st, max(3, min(steps, 5)), 1, world)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        from tools import cpu_ref as CR
        cpu = CR.c2_baseline(T, args.sampler, noise_mode, CR.host_cores(),
                             target_s=3.0 if headline else 1.5)
    sampler_name = {0: "seq", 1: "prefix", 2: "dnc"}[st["sampler"]]
    rec = {
        "value": value, "unit": UNIT, "ms_per_step": ms / steps, "steps": steps,
        "warmup": args.warmup,
        "config": {"workload": f"C2: lgssm-synthetic d=4 dy=1 T={T}, {C} chains/GPU, "
                               f"pit::{sampler_name}_sample from one shared Kalman filter",
                   "noise": noise_mode, "chains_per_gpu": C, "T": T,
                   "parallelism": f"chains sharded over {world} GPU(s)",
                   "l2": "inputs+outputs (4.3 GB) >> L2 (126 MB); no flush needed",
                   "mcmc_sweeps_per_sec": 1e3 * steps / ms},
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if check is not None:
        rec["spot_check"] = check
    return rec


# ---------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU implementation (oracle/_ref) of the
    headline workload on all host cores, rank 0 only: pit::prefix_sample per chain
    from one shared kalman_filter result, variates pre-drawn and read through a
    NoiseSource (the GPU arm's noise mode), each step a bounded sample of chains."""
    if rank != 0:
        return
    from tools import cpu_ref as CR
    T = args.T or 65536
    threads = CR.host_cores()
    ref = CR.C2Ref(T, 4, args.sampler, args.noise, n_noise=min(threads, 4))
    _, t1 = ref.run(1, 1)
    per_step = threads * max(1, int(round(1.5 / max(t1, 1e-3))))
    for _ in range(min(args.warmup, 1)):
        ref.run(threads, threads)
    secs = 0.0
    for _ in range(args.steps):
        _, dt = ref.run(per_step, threads)
        secs += dt
    value = per_step * (T + 1) * args.steps / secs
    sample = (f"{per_step} chains x (T+1)={T + 1} per step, pit::{args.sampler}_sample "
              f"({args.noise} variates), {threads} threads")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": f"C2: lgssm-synthetic d=4 dy=1 T={T}, pit::{args.sampler}_sample "
                               f"per chain from one shared Kalman filter, on host cores",
                   "noise": args.noise, "chains_per_step": per_step, "T": T,
                   "implementation": "oracle/_ref: unmodified /root/reference/proj/src built "
                                     "against the Eigen shim" if ref.kind == "reference"
                                     else "oracle/ C restatement (port)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": ref.kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- main
def line_from(rec, args, world, scaling="weak"):
    line = {"metric": METRIC, "value": rec["value"], "unit": UNIT, "n_gpus": world,
            "steps": rec["steps"], "warmup": rec.get("warmup", args.warmup),
            "ms_per_step": rec["ms_per_step"], "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic"}
    for k in ("config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks", "spot_check"):
        if k in rec:
            line[k] = rec[k]
    return line


def main():
    args = parse()
    if args.impl == "b200":
        maybe_self_launch(args)
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    from paper_2303_00301_b200 import _lib
    torch.cuda.set_device(local)
    if _lib.load().auxmc_device_ok() != 1:
        raise SystemExit("libauxmc_b200: no usable sm_100 device")
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    try:
        from tools import bench_aux
        if args.config in ("all", "c2"):
            rec = run_c2(args, rank, world, local, args.noise)
            line = line_from(rec, args, world)
            if args.config == "all" and not args.no_configs:
                configs = {}
                if args.noise == "predrawn":
                    configs["c2_rng"] = run_c2(args, rank, world, local, "rng", args.min_time,
                                               headline=False)
                for name in ("c1", "c3", "c4", "c4_1chain", "c5"):
                    if world == 1:  # one failing sub-record must not cost the headline line
                        try:
                            configs[name] = bench_aux.record(name, args, rank, world, local)
                        except Exception as e:  # noqa: BLE001 - reported in the line
                            configs[name] = {"error": f"{type(e).__name__}: {e}"[:300]}
                            try:
                                torch.cuda.synchronize()
                            except Exception:  # noqa: BLE001 - a sticky context error
                                pass
                    else:  # ranks fail together (torchrun tears the job down): no hang
                        configs[name] = bench_aux.record(name, args, rank, world, local)
                line["configs"] = configs
                # launches of every config's timed region count as ours too
                line["gpu_launches_all_configs"] = line["gpu_launches"] + sum(
                    c.get("gpu_launches", 0) for c in configs.values())
        elif args.config == "c5ts":
            rec = bench_aux.record("c5ts", args, rank, world, local)
            line = line_from(rec, args, world, scaling="strong")
        else:
            rec = bench_aux.record(args.config, args, rank, world, local)
            line = line_from(rec, args, world)
        if rank == 0:
            print(json.dumps(line), flush=True)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
