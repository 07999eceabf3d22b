"""N > 1 path on CPU: world-size-2 gloo run of the chain sharding.

Chains are independent; a chain is identified by its global index only
(root = from_seed(seed).derive(kChain, c), runner.cpp:132), so a sharded run
must reproduce the single-process run chain for chain, with no collective on
the data path.  The worker (tests/mp/shard_worker.py) runs under
torch.distributed.run exactly as bench.py does on GPUs, with gloo instead of NCCL.
"""
import json
import socket
import subprocess
import sys

import numpy as np

from conftest import ROOT


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_weak_and_strong_shards():
    from paper_2303_00301_b200 import shard
    assert [shard.weak_shard(r, 4, 3).first for r in range(4)] == [0, 3, 6, 9]
    for total in (0, 1, 5, 8, 13):
        for world in (1, 2, 3, 8):
            parts = [shard.strong_shard(r, world, total) for r in range(world)]
            idx = [i for p in parts for i in range(p.first, p.first + p.count)]
            assert idx == list(range(total))
            assert max(p.count for p in parts) - min(p.count for p in parts) <= 1


def test_world2_gloo_sharding_matches_single_process(tmp_path, oracle):
    out = tmp_path / "mp.json"
    per_rank, steps = 2, 3
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           str(ROOT / "tests" / "mp" / "shard_worker.py"), str(out), str(per_rank), str(steps)]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    res = json.load(open(out))
    assert res["world"] == 2
    # keys: the sharded gather equals the single-process derivation
    root = oracle.from_seed(7)
    want_keys = [int(oracle.derive(root, oracle.L_CHAIN, c).key) for c in range(2 * per_rank)]
    assert res["keys"] == want_keys
    # paths: the sharded chains equal a single-process run over all chains
    s = oracle.spec("lgssm-synthetic", T=12, dx=2, dy=1, data_seed=3)
    _, data = oracle.simulate(s)
    tg = oracle.make_target(s, data)
    x0 = np.tile(tg.arrays()["m0"], (13, 1))
    for c in range(2 * per_rank):
        ch = oracle.AuxChain(tg, x0, 0.6)
        for _ in range(steps):
            ch.step(oracle.derive(root, oracle.L_CHAIN, c), 0)
        assert np.array_equal(np.asarray(res["paths"][c]), ch.x), f"chain {c}"
    assert res["tmax"] == 2.5  # max over ranks of 1.5 + rank
    assert [(p["first"], p["count"]) for p in res["strong"]] == [(0, 3), (3, 2)]
