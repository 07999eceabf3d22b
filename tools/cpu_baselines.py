"""CPU reference timings for BASELINE.md §5 (oracle port of the reference
algorithm, -O2 C, this host): one core, bounded samples, chain-timesteps/s.

usage: python tools/cpu_baselines.py [--threads N] > profiles/r1_cpu_baselines.json
The oracle is the C restatement in oracle/ (test infrastructure); a compiled
reference is not available (Eigen absent), so kind = "port".
"""
import argparse
import concurrent.futures as cf
import json
import os
import pathlib
import platform
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from oracle import pyoracle as O  # noqa: E402


def timed(fn, n_workers, n_items):
    t0 = time.perf_counter()
    if n_workers == 1:
        for i in range(n_items):
            fn(i)
    else:
        with cf.ThreadPoolExecutor(max_workers=n_workers) as ex:
            list(ex.map(fn, range(n_items)))
    return time.perf_counter() - t0


def aux_config(kind, T, delta, backend, pf, steps, **kw):
    s = O.spec(kind, T=T, **kw)
    lat, data = O.simulate(s)
    tg = O.make_target(s, data)
    x0 = lat if kind != "lgssm-synthetic" else np.tile(tg.arrays()["m0"], (T + 1, 1))

    def run(c):
        ch = O.AuxChain(tg, x0, delta)
        root = O.derive(O.from_seed(1), O.L_CHAIN, c)
        for _ in range(steps):
            ch.step(root, backend, pf)
    return run


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    O.build()
    out = {"host": platform.processor() or platform.machine(), "nproc": os.cpu_count(),
           "kind": "port", "rows": []}

    def row(name, ct_per_item, fn, items, workers, note):
        dt = timed(fn, workers, items)
        out["rows"].append({"config": name, "cores": workers, "items": items,
                            "seconds": dt, "value": ct_per_item * items / dt,
                            "unit": "chain-timesteps/s", "sample": note})
        print(json.dumps(out["rows"][-1]), file=sys.stderr, flush=True)

    # C1: one chain, T = 1024, prefix backend with the scan filter, 20 iterations
    row("C1", 1025 * 20, aux_config("lgssm-synthetic", 1024, 1.0, 1, 1, 20, dx=1, dy=1,
                                      data_seed=1), 1, 1, "1 chain x 20 iterations, T=1024")
    # C2: prefix_sample per chain, T = 2^16, d = 4
    s = O.spec("lgssm-synthetic", T=65536, dx=4, dy=1, data_seed=1)
    lat, data = O.simulate(s)
    m = O.synthetic_lgssm(s)
    fr = O.kalman_filter(m, data)
    for name, fnc in (("C2 prefix", O.prefix_sample), ("C2 DnC", O.dnc_sample)):
        f = (lambda fnc: lambda c: fnc(m, fr, O.stream_noise(O.derive(O.from_seed(1), O.L_CHAIN, c))))(fnc)
        row(name, 65537, f, 2, 1, "2 chains, T=65536, 1 core")
        row(name, 65537, f, 2 * a.threads, a.threads, f"{2 * a.threads} chains, {a.threads} threads")
    # C3: Lorenz-96 d = 40, T = 4096, sequential backend, 1 iteration per chain
    f3 = aux_config("lorenz96", 4096, 0.05, 0, 0, 1, dx=40, data_seed=3)
    row("C3", 4097, f3, 1, 1, "1 chain x 1 iteration, T=4096")
    row("C3", 4097, f3, a.threads, a.threads, f"{a.threads} chains x 1 iteration")
    # C4: reference cSMC, N = 256, T = 2^14, 1 iteration
    s4 = O.spec("stochvol", T=16384, dx=3, data_seed=11)
    lat4, data4 = O.simulate(s4)
    tg4 = O.make_target(s4, data4)

    def f4(c):
        pg = O.PGChain(tg4, lat4, 1.0)
        pg.step(256, O.derive(O.from_seed(1), O.L_CHAIN, c), 1)
    row("C4 ref-cSMC", 16385, f4, 1, 1, "1 chain x 1 iteration, N=256, T=16384")
    row("C4 ref-cSMC", 16385, f4, a.threads, a.threads, f"{a.threads} chains x 1 iteration")
    # C5: spatio-temporal grid 4 at T = 2^14 (extrapolated linearly to 2^20)
    f5 = aux_config("spatio-temporal", 16384, 0.5, 1, 1, 1, grid=4, data_seed=7)
    row("C5 (T=2^14, extrapolate)", 16385, f5, 1, 1, "1 chain x 1 iteration, T=16384")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
