"""Time-sharded scan filter and prefix sampler: pit::parallel_filter
(pit.cpp:117-188) and pit::prefix_sample (pit.cpp:78-115) for one long sequence
split over ranks.

The horizon's block tree (blocks of LB steps, super-blocks of SB = LB² steps)
depends only on T.  Rank r owns a contiguous run of super-blocks
(`shard.strong_shard` over the super-block count); the only exchange is one
all-gather of the super-block aggregates (the filtering-element tuple
(A, b, C, η, J), 3d² + 2d doubles each) and one of the per-super-block
log-likelihood partials.  Every rank count reproduces one rank bit for bit.

`exchange` is any all-gather of equally shaped device tensors in rank order:
`torch.distributed.all_gather` under NCCL (ranks on their own GPUs) or gloo (host
tensors), or `LocalExchange` to run several shards in one process.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib
from .lgssm import FilterResult, Model, _dev, _stream
from .shard import strong_shard


@dataclass(frozen=True)
class TShardGeom:
    T: int
    LB: int
    nblk: int
    nsup: int
    SB: int
    elem_doubles: int

    @staticmethod
    def of(T: int, dx: int) -> "TShardGeom":
        v = [C.c_int() for _ in range(5)]
        _lib.check(_lib.load().auxmc_tshard_geometry(T, dx, *[C.byref(x) for x in v]),
                   "tshard_geometry")
        return TShardGeom(T, *[x.value for x in v])

    def owned(self, rank: int, world: int):
        """Super-block range [lo, hi) and time range [t_lo, t_hi) of a rank."""
        sh = strong_shard(rank, world, self.nsup)
        lo, hi = sh.first, sh.first + sh.count
        return lo, hi, min(lo * self.SB, self.T + 1), min(hi * self.SB, self.T + 1)


def torch_exchange(group=None):
    """All-gather through torch.distributed (NCCL device tensors or gloo host tensors)."""
    import torch.distributed as dist

    def ex(t: torch.Tensor) -> list:
        backend = dist.get_backend(group)
        x = t if backend == "nccl" else t.cpu()
        parts = [torch.empty_like(x) for _ in range(dist.get_world_size(group))]
        dist.all_gather(parts, x.contiguous(), group=group)
        return [p.to(t.device) for p in parts]
    return ex


class ShardedScanFilter:
    """One rank's share of the scan filter of `obs` ([T+1, dy]) under `model`."""

    def __init__(self, model: Model, rank: int, world: int):
        self.model, self.rank, self.world = model, rank, world
        self.geom = TShardGeom.of(model.T, model.dx)
        self.sup_lo, self.sup_hi, self.t_lo, self.t_hi = self.geom.owned(rank, world)
        lib = _lib.load()
        self._mr = model.raw()
        self.ws_bytes = lib.auxmc_tshard_filter_workspace(C.byref(self._mr))
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=model.device)
        self.max_owned = -(-self.geom.nsup // world)  # ceil: rows each rank contributes

    def local(self, obs) -> torch.Tensor:
        """Phase 1: this rank's super-block aggregates, padded to max_owned rows.
        `obs` is a [T+1, dy] array or a device pointer (int) to one."""
        g, dev = self.geom, self.model.device
        if isinstance(obs, int):
            self.obs, self._obs_ptr = None, obs
        else:
            self.obs = _dev(obs, dev).contiguous()
            self._obs_ptr = self.obs.data_ptr()
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        out = torch.zeros((self.max_owned, g.elem_doubles), dtype=torch.float64, device=dev)
        if self.sup_hi > self.sup_lo:
            _lib.check(_lib.load().auxmc_tshard_filter_local(
                C.byref(self._mr), self._obs_ptr, self.sup_lo, self.sup_hi,
                self.ws.data_ptr(), self.ws_bytes, out.data_ptr(), self.status.data_ptr(),
                _stream()), "tshard_filter_local")
        return out

    def _concat(self, parts, rows_of):
        return torch.cat([p[:rows_of(r)] for r, p in enumerate(parts)], 0).contiguous()

    def _rows(self, r):
        lo, hi, _, _ = self.geom.owned(r, self.world)
        return hi - lo

    def finish(self, gathered_aggs, fr: FilterResult | None = None):
        """Phase 2 (after the all-gather): moments for this rank's time range and its
        log-likelihood partials (padded to max_owned)."""
        g, dev = self.geom, self.model.device
        sup_all = self._concat(gathered_aggs, self._rows)
        assert sup_all.shape[0] == g.nsup
        if fr is None:
            fr = FilterResult.empty(1, g.T, self.model.dx, dev)
        ll = torch.zeros(self.max_owned, dtype=torch.float64, device=dev)
        if self.sup_hi > self.sup_lo:
            raw = fr.raw()
            _lib.check(_lib.load().auxmc_tshard_filter_finish(
                C.byref(self._mr), self._obs_ptr, self.sup_lo, self.sup_hi,
                self.ws.data_ptr(), self.ws_bytes, sup_all.data_ptr(), C.byref(raw),
                ll.data_ptr(), self.status.data_ptr(), _stream()), "tshard_filter_finish")
        return fr, ll

    def log_marginal(self, gathered_ll) -> torch.Tensor:
        """Sum of every super-block partial in super-block order (device scalar)."""
        parts = self._concat(gathered_ll, self._rows)
        out = torch.empty(1, dtype=torch.float64, device=self.model.device)
        _lib.check(_lib.load().auxmc_tshard_sum(parts.data_ptr(), parts.numel(), out.data_ptr(),
                                                 _stream()), "tshard_sum")
        return out


def sharded_filter(model: Model, obs, rank: int, world: int, exchange):
    """Run the time-sharded scan filter; returns (FilterResult with this rank's time
    range filled, log_marginal, (t_lo, t_hi))."""
    sf = ShardedScanFilter(model, rank, world)
    aggs = sf.local(obs)
    fr, ll = sf.finish(exchange(aggs))
    lm = sf.log_marginal(exchange(ll))
    fr.log_marginal.copy_(lm)
    return fr, lm, (sf.t_lo, sf.t_hi)


class ShardedPrefixSampler:
    """One rank's share of pit::prefix_sample for one path, on the time range of its
    ShardedScanFilter (same super-blocks)."""

    def __init__(self, sf: ShardedScanFilter):
        self.sf, self.model = sf, sf.model
        lib = _lib.load()
        Lb, P = C.c_int(), C.c_int()
        _lib.check(lib.auxmc_tshard_prefix_geometry(self.model.T, C.byref(Lb), C.byref(P)),
                   "tshard_prefix_geometry")
        self.Lb, self.P = Lb.value, P.value
        if sf.geom.SB % self.Lb:
            raise ValueError("sampler blocks must divide the filter super-blocks")
        self.ws_bytes = lib.auxmc_tshard_prefix_workspace(C.byref(sf._mr))
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.model.device)
        self.rows = self.model.dx * self.model.dx + self.model.dx
        self.max_blocks = max(1, (sf.geom.SB // self.Lb) * sf.max_owned)  # rows per rank

    def _blocks(self, r):
        _, _, t_lo, t_hi = self.sf.geom.owned(r, self.sf.world)
        s_hi = min(t_hi, self.model.T)
        return (t_lo // self.Lb, -(-s_hi // self.Lb)) if s_hi > t_lo else (0, 0)

    def local(self, fr: FilterResult, noise, traj: torch.Tensor):
        """Phase 1: block rows of this rank (padded) and x_T (zeros unless this rank owns T)."""
        dev, d = self.model.device, self.model.dx
        self.noise_raw = noise.raw()
        k_lo, k_hi = self._blocks(self.sf.rank)
        out = torch.zeros((self.max_blocks, self.rows), dtype=torch.float64, device=dev)
        xT = torch.zeros(d, dtype=torch.float64, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        if self.sf.t_hi > self.sf.t_lo:
            raw = fr.raw()
            _lib.check(_lib.load().auxmc_tshard_prefix_local(
                C.byref(self.sf._mr), C.byref(raw), C.byref(self.noise_raw), self.sf.t_lo,
                self.sf.t_hi, self.ws.data_ptr(), self.ws_bytes, out.data_ptr(), xT.data_ptr(),
                traj.data_ptr(), self.status.data_ptr(), _stream()), "tshard_prefix_local")
        return out, xT

    def finish(self, gathered_rows, gathered_xT, traj: torch.Tensor):
        """Phase 2: the path on this rank's time range (written into traj [T+1, d])."""
        parts = []
        for r, p in enumerate(gathered_rows):
            k_lo, k_hi = self._blocks(r)
            parts.append(p[:k_hi - k_lo])
        blk_all = torch.cat(parts, 0).contiguous()
        assert blk_all.shape[0] == self.P, (blk_all.shape, self.P)
        owner = next(r for r in range(self.sf.world)
                     if self.sf.geom.owned(r, self.sf.world)[2] < self.model.T + 1 ==
                     self.sf.geom.owned(r, self.sf.world)[3])
        xT = gathered_xT[owner].contiguous()
        if self.sf.t_hi > self.sf.t_lo:
            _lib.check(_lib.load().auxmc_tshard_prefix_finish(
                C.byref(self.sf._mr), C.byref(self.noise_raw), self.sf.t_lo, self.sf.t_hi,
                self.ws.data_ptr(), self.ws_bytes, blk_all.data_ptr(), xT.data_ptr(),
                traj.data_ptr(), _stream()), "tshard_prefix_finish")
        else:  # a rank that owns no super-block still gets row T
            traj[self.model.T].copy_(xT)
        return traj


def sharded_filter_and_prefix(model: Model, obs, noise, rank: int, world: int, exchange):
    """Scan filter + prefix path of one sequence split over ranks; returns
    (FilterResult, log_marginal, traj [T+1, d], (t_lo, t_hi)) with this rank's time
    range filled (traj row T on every rank)."""
    sf = ShardedScanFilter(model, rank, world)
    fr, ll = sf.finish(exchange(sf.local(obs)))
    lm = sf.log_marginal(exchange(ll))
    fr.log_marginal.copy_(lm)
    ps = ShardedPrefixSampler(sf)
    traj = torch.zeros((model.T + 1, model.dx), dtype=torch.float64, device=model.device)
    rows, xT = ps.local(fr, noise, traj)
    ps.finish(exchange(rows), exchange(xT), traj)
    return fr, lm, traj, (sf.t_lo, sf.t_hi)


class LocalExchange:
    """Runs `world` shards in one process: collects each shard's tensor, then hands
    every shard the rank-ordered list (for tests and single-GPU checks)."""

    @staticmethod
    def run(model: Model, obs, world: int, noise=None):
        shards = [ShardedScanFilter(model, r, world) for r in range(world)]
        aggs = [s.local(obs) for s in shards]
        outs = [s.finish(aggs) for s in shards]
        lls = [ll for _, ll in outs]
        lm = shards[0].log_marginal(lls)
        frs = [fr for fr, _ in outs]
        if noise is None:
            return shards, frs, lm
        samplers = [ShardedPrefixSampler(s) for s in shards]
        trajs = [torch.zeros((model.T + 1, model.dx), dtype=torch.float64, device=model.device)
                 for _ in shards]
        loc = [p.local(fr, noise, tr) for p, fr, tr in zip(samplers, frs, trajs)]
        rows = [r for r, _ in loc]
        xts = [x for _, x in loc]
        for p, tr in zip(samplers, trajs):
            p.finish(rows, xts, tr)
        return shards, frs, lm, trajs


class RawModel:
    """An auxmc_lgssm struct produced by the library (device pointers), with the
    attributes the sharded scans read."""

    def __init__(self, raw, device):
        self._raw, self.device = raw, device
        self.T, self.dx, self.dy = raw.T, raw.dx, raw.dy

    def raw(self):
        return self._raw


class _KeyNoise:
    """Stream noise keyed by one device key (the iteration key of the aux step)."""

    def __init__(self, key_ptr: int):
        self.key_ptr = key_ptr

    def raw(self):
        n = _lib.Noise()
        n.kind = _lib.NOISE_STREAM
        n.keys = self.key_ptr
        return n


class ShardedAuxChain:
    """One chain's auxiliary Kalman step (auxk::kernel_step, prefix backend, scan
    filter) with the horizon split over ranks.  Rank r works only on
    its own time range [t_lo, t_hi) of whole filter super-blocks (plus one halo row on
    each side): aux observations, surrogate models, path log-densities, log gamma,
    gradients, the two sharded filters and the sharded prefix draw.  Per step the ranks
    exchange the filters' super-block aggregates and log-likelihood partials, the
    sampler's block rows, the proposal's halo rows (2 d doubles per rank) and the step's
    super-block partials with the status flags (6 doubles per super-block) — never a
    path.  Every split gives the same bits (tests/test_gpu_tshard_aux.py)."""

    def __init__(self, chains, rank: int, world: int, exchange, zeroth_order=False):
        if chains.C != 1:
            raise ValueError("ShardedAuxChain: one chain")
        self.ch, self.rank, self.world, self.exchange = chains, rank, world, exchange
        self.tg = chains.target
        self.opts = _lib.KernelOptions(1, 1, int(zeroth_order))  # prefix, scan filter
        lib = _lib.load()
        self._tr = self.tg.raw()
        self.ws_bytes = lib.auxmc_tshard_aux_workspace(C.byref(self._tr))
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.tg.device)
        self.geom = TShardGeom.of(self.tg.T, self.tg.dx)
        self.sup_lo, self.sup_hi, self.t_lo, self.t_hi = self.geom.owned(rank, world)
        self.max_owned = -(-self.geom.nsup // world)
        self.traj = torch.zeros((self.tg.T + 1, self.tg.dx), dtype=torch.float64,
                                device=self.tg.device)

    def _halo(self, traj):
        """x'_{t_lo-1} and x'_{t_hi} from the neighbours (every rank sends its first and
        last own rows)."""
        d, dev = self.tg.dx, self.tg.device
        lo, hi = self.t_lo, self.t_hi
        edge = torch.zeros((2, d), dtype=torch.float64, device=dev)
        if hi > lo:
            edge[0] = traj[lo]
            edge[1] = traj[hi - 1]
        parts = self.exchange(edge)
        if hi <= lo:
            return
        if lo > 0:
            prev = max(r for r in range(self.rank) if self.geom.owned(r, self.world)[3] >
                       self.geom.owned(r, self.world)[2])
            traj[lo - 1] = parts[prev][1]
        if hi <= self.tg.T:
            nxt = min(r for r in range(self.rank + 1, self.world)
                      if self.geom.owned(r, self.world)[3] > self.geom.owned(r, self.world)[2])
            traj[hi] = parts[nxt][0]

    def step(self):
        lib, dev = _lib.load(), self.tg.device
        T, d = self.tg.T, self.tg.dx
        ch = self.ch.raw()
        model = _lib.Lgssm()
        z, prop, it = C.c_void_p(), C.c_void_p(), C.c_void_p()
        lo, hi = self.t_lo, self.t_hi
        _lib.check(lib.auxmc_tshard_aux_begin(
            C.byref(self._tr), C.byref(ch), C.byref(self.opts), self.ws.data_ptr(),
            self.ws_bytes, lo, hi, C.byref(model), C.byref(z), C.byref(prop), C.byref(it),
            _stream()), "tshard_aux_begin")
        rm = RawModel(model, dev)
        # forward filter and the path draw, time-sharded
        sf = ShardedScanFilter(rm, self.rank, self.world)
        fr, ll = sf.finish(self.exchange(sf.local(z.value)))
        lm_fwd = sf.log_marginal(self.exchange(ll))
        fr.log_marginal.copy_(lm_fwd)
        ps = ShardedPrefixSampler(sf)
        traj = self.traj
        rows, xT = ps.local(fr, _KeyNoise(it.value), traj)
        ps.finish(self.exchange(rows), self.exchange(xT), traj)
        self._halo(traj)
        if hi > lo:
            h0, h1 = max(lo - 1, 0), min(hi + 1, T + 1)
            _lib.check(lib.auxmc_copy_device(prop.value + h0 * d * 8, traj[h0:h1].data_ptr(),
                                             (h1 - h0) * d * 8, _stream()), "copy")
        part = torch.zeros((self.max_owned + 2, 5), dtype=torch.float64, device=dev)
        flags = torch.zeros(8, dtype=torch.int32, device=dev)
        flags[0] = sf.status[0]
        flags[1] = ps.status[0]
        _lib.check(lib.auxmc_tshard_aux_middle(
            C.byref(self._tr), C.byref(ch), C.byref(self.opts), self.ws.data_ptr(),
            self.ws_bytes, lo, hi, part.data_ptr(), flags.data_ptr(), _stream()),
            "tshard_aux_middle")
        # reverse filter on the surrogate at x'
        sr = ShardedScanFilter(rm, self.rank, self.world)
        _, llr = sr.finish(self.exchange(sr.local(z.value)))
        lm_rev = sr.log_marginal(self.exchange(llr))
        flags[5] = sr.status[0]
        _lib.check(lib.auxmc_tshard_aux_end(
            C.byref(self._tr), C.byref(ch), C.byref(self.opts), self.ws.data_ptr(),
            self.ws_bytes, lo, hi, part.data_ptr(), flags.data_ptr(), _stream()),
            "tshard_aux_end")
        # one exchange: super-block partials (rows 0..owned) with the flags in the last row
        part[self.max_owned + 1, :].zero_()
        part[self.max_owned, :] = 0.0
        part[self.max_owned, 0:5] = flags[0:5].to(torch.float64)
        part[self.max_owned + 1, 0:2] = flags[5:7].to(torch.float64)
        parts = self.exchange(part)
        rows_all, fl = [], torch.zeros(8, dtype=torch.float64, device=dev)
        for r, pr in enumerate(parts):
            s_lo, s_hi, _, _ = self.geom.owned(r, self.world)
            rows_all.append(pr[:s_hi - s_lo])
            fl[0:5] = torch.maximum(fl[0:5], pr[self.max_owned, 0:5])
            fl[5:7] = torch.maximum(fl[5:7], pr[self.max_owned + 1, 0:2])
        parts_all = torch.cat(rows_all, 0).contiguous()
        flags_all = fl.to(torch.int32).contiguous()
        _lib.check(lib.auxmc_tshard_aux_decide(
            C.byref(self._tr), C.byref(ch), self.ws.data_ptr(), self.ws_bytes, lo, hi,
            parts_all.data_ptr(), parts_all.shape[0], lm_fwd.data_ptr(), lm_rev.data_ptr(),
            flags_all.data_ptr(), _stream()), "tshard_aux_decide")


class LocalShardedAux:
    """Runs `world` ShardedAuxChain ranks in one process (tests): each rank owns
    its own chain state copy; every exchange is served once all ranks posted."""

    @staticmethod
    def assemble(chains) -> torch.Tensor:
        """The chain's full path from the ranks' own time ranges (a rank's state is
        valid on its range and one halo row on each side only)."""
        world = len(chains)
        T, d = chains[0].target.T, chains[0].target.dx
        geom = TShardGeom.of(T, d)
        out = torch.empty((1, T + 1, d), dtype=torch.float64, device=chains[0].x.device)
        for r, ch in enumerate(chains):
            _, _, lo, hi = geom.owned(r, world)
            out[0, lo:hi] = ch.x[0, lo:hi]
        return out

    @staticmethod
    def run(make_chains, world: int, steps: int):
        return LocalShardedAux.run_on([make_chains() for _ in range(world)], steps)

    @staticmethod
    def run_on(chains, steps: int):
        """Continue `len(chains)` rank states for `steps` more sharded steps."""
        import threading
        world = len(chains)
        barrier = threading.Barrier(world)
        box = {}
        lock = threading.Lock()
        errors = []

        def make_ex(rank):
            seq = [0]

            def ex(t):
                k = seq[0]
                seq[0] += 1
                torch.cuda.synchronize()
                with lock:
                    box.setdefault(k, [None] * world)[rank] = t.clone()
                barrier.wait()
                out = [x.to(t.device) for x in box[k]]
                barrier.wait()
                return out
            return ex

        def worker(r):
            try:
                sa = ShardedAuxChain(chains[r], r, world, make_ex(r))
                for _ in range(steps):
                    sa.step()
                torch.cuda.synchronize()
            except Exception as e:  # noqa: BLE001
                errors.append(e)
                barrier.abort()

        th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if errors:
            raise errors[0]
        return chains
