"""One rank of the world-size-2 sharding test (launched by tests/test_multiproc.py
through torch.distributed.run with the gloo backend, on CPU).

Each rank takes its weak-scaling shard of chains, derives the chain roots with
the product's host RNG, runs the oracle auxiliary Kalman step on its own chains
only (the CPU stand-in for the per-GPU work), and gathers keys, paths and the
max-over-ranks timing reduction the bench uses.  Rank 0 writes the result.
"""
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main(out_path, per_rank, steps):
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    from paper_2303_00301_b200 import rng, shard
    from oracle import pyoracle as O
    sh = shard.weak_shard(rank, world, per_rank)
    keys = rng.chain_keys(7, sh.count, first=sh.first, device="cpu")
    all_keys = shard.gather_rows(keys, world)

    s = O.spec("lgssm-synthetic", T=12, dx=2, dy=1, data_seed=3)
    _, data = O.simulate(s)
    tg = O.make_target(s, data)
    x0 = np.tile(tg.arrays()["m0"], (13, 1))
    root = O.from_seed(7)
    xs = []
    for c in range(sh.first, sh.first + sh.count):
        ch = O.AuxChain(tg, x0, 0.6)
        for _ in range(steps):
            ch.step(O.derive(root, O.L_CHAIN, c), 0)
        xs.append(ch.x)
    paths = shard.gather_rows(torch.from_numpy(np.stack(xs)), world)
    tmax = shard.max_over_ranks(1.5 + rank, world)
    strong = [shard.strong_shard(rank, world, 5).__dict__]
    gathered = [None] * world
    dist.all_gather_object(gathered, strong[0])
    if rank == 0:
        json.dump({"keys": [int(k) for k in all_keys.numpy().view(np.uint64)],
                   "paths": paths.numpy().tolist(), "tmax": tmax, "strong": gathered,
                   "world": world}, open(out_path, "w"))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]))
