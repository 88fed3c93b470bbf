"""Sharded (multi-GPU) HistoCore and PeelOne drivers -- SURVEY 8(e), 8(f)
NEXT-1; PAPER.md P:894 lists multi-GPU as future work.

The compute of every step runs in libpico's kernels (include/pico_shard.h).
This module is the plumbing between the steps:
  * the arc-balanced 1-D vertex partition;
  * the exchange: all-gather of the per-rank counts (which is also the global
    convergence test: a round with a global count of 0 ends the run) and an
    all-gather(v) of the changed (v, oldcore, core) triples;
  * the round loop (HistoCore) / the level and sub-round loops (PeelOne:
    an all-gather of (|F|, kmin) pairs and an all-gatherv of F per sub-round).

Exchanges:
  * TorchDistExchange -- torch.distributed (NCCL over NVLink/NVSwitch on B200,
    gloo on CPU for the host-logic tests), one process per GPU;
  * loopback -- P logical shards in one process on one GPU, the all-gather is
    a device concatenation (coreness_loopback); this is how the sharded kernels
    are parity-tested on a single GPU.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from ._lib import check, load


# ---------------------------------------------------------------------------
# partition (host logic)
# ---------------------------------------------------------------------------
def partition(rowptr, nparts: int) -> list[int]:
    """Vertex boundaries [b_0 = 0, b_1, ..., b_P = n] of contiguous ranges
    with ~2m/P arcs each: b_r = first v with rowptr[v] >= r * 2m / P."""
    rp = np.asarray(rowptr if not hasattr(rowptr, "cpu") else rowptr.cpu().numpy(), dtype=np.int64)
    n = rp.size - 1
    arcs = int(rp[-1])
    bounds = [0]
    for r in range(1, nparts):
        target = (arcs * r) // nparts
        b = int(np.searchsorted(rp, target, side="left"))
        bounds.append(min(max(b, bounds[-1]), n))
    bounds.append(n)
    return bounds


def partition_vertices(n: int, nparts: int) -> list[int]:
    """Equal vertex ranges [n r / P, n (r+1) / P): the partition of a run whose
    ranks generate only their own rows (no global rowptr to balance arcs on;
    the generators' seeded relabel spreads the hubs, so the ranges' arc counts
    are balanced in expectation)."""
    return [n * r // nparts for r in range(nparts + 1)]


def local_rows(rowptr, colidx, vb: int, ve: int):
    """Rows [vb, ve) as (rowptr_local with rowptr_local[0] = 0, colidx_local)."""
    a, b = int(rowptr[vb]), int(rowptr[ve])
    rp = rowptr[vb:ve + 1] - a
    return rp.contiguous(), colidx[a:b].contiguous()


# ---------------------------------------------------------------------------
# exchanges
# ---------------------------------------------------------------------------
class TorchDistExchange:
    """allgather / allgatherv over a torch.distributed process group."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def allgather_counts(self, count: int, device) -> list[int]:
        import torch
        t = torch.tensor([count], dtype=torch.int64, device=device)
        out = torch.empty(self.world, dtype=torch.int64, device=device)
        self.dist.all_gather_into_tensor(out, t, group=self.group)
        return out.tolist()  # one host read for all ranks

    def allgatherv(self, local, counts: list[int]):
        """Concatenation in rank order of every rank's `local[:counts[rank]]`
        (1-D tensors); all-gather of max-padded buffers."""
        import torch
        mx = max(counts)
        if mx == 0:
            return local[:0]
        buf = torch.zeros(mx, dtype=local.dtype, device=local.device)
        buf[:counts[self.rank]] = local[:counts[self.rank]]
        out = torch.empty(self.world * mx, dtype=local.dtype, device=local.device)
        self.dist.all_gather_into_tensor(out, buf, group=self.group)
        if all(c == mx for c in counts):
            return out
        return torch.cat([out[r * mx:r * mx + c] for r, c in enumerate(counts)])

    def allgather_pairs(self, a: int, b: int, device) -> list[tuple[int, int]]:
        """Every rank's (a, b), in rank order (one collective)."""
        import torch
        t = torch.tensor([a, b], dtype=torch.int64, device=device)
        out = torch.empty(2 * self.world, dtype=torch.int64, device=device)
        self.dist.all_gather_into_tensor(out, t, group=self.group)
        v = out.tolist()
        return [(v[2 * r], v[2 * r + 1]) for r in range(self.world)]

    def max_over_ranks(self, x: float, device) -> float:
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())


# ---------------------------------------------------------------------------
# one rank's shard (ctypes wrapper of pico_shard_*)
# ---------------------------------------------------------------------------
class DeviceShard:
    """The rank's state in libpico (owned rows [vb, vb + nloc))."""

    def __init__(self, rowptr_local, colidx_local, vb: int, n_global: int, flags: int = 0, stream=None):
        import torch
        self.lib = load()
        self.dev = rowptr_local.device
        self.rp, self.ci = rowptr_local, colidx_local  # kept alive for the handle
        self.nloc = rowptr_local.numel() - 1
        self.vb, self.n_global = vb, n_global
        self.stream = stream or torch.cuda.current_stream(self.dev)
        h = ctypes.c_void_p()
        check(self.lib.pico_shard_create(self.rp.data_ptr(), self.ci.data_ptr() if self.ci.numel() else None,
                                         self.nloc, vb, n_global, flags, ctypes.c_void_p(self.stream.cuda_stream),
                                         ctypes.byref(h)))
        self.h = h
        self.trip = torch.empty(3 * max(self.nloc, 1), dtype=torch.int32, device=self.dev)

    def degrees(self):
        import torch
        d = torch.empty(max(self.nloc, 1), dtype=torch.int32, device=self.dev)
        check(self.lib.pico_shard_degrees(self.h, d.data_ptr()))
        return d[:self.nloc]

    def init(self, deg_global) -> int:
        c = ctypes.c_int64()
        check(self.lib.pico_shard_init(self.h, deg_global.data_ptr(), ctypes.byref(c)))
        return c.value

    def pack(self):
        c = ctypes.c_int64()
        check(self.lib.pico_shard_pack(self.h, self.trip.data_ptr(), self.trip.numel() // 3, ctypes.byref(c)))
        return self.trip, c.value

    def apply(self, triples, total: int, wait: bool = False):
        """Asynchronous unless wait=True (then returns |C_{t+1}| of this rank)."""
        if not wait:
            check(self.lib.pico_shard_apply(self.h, triples.data_ptr() if total else None, total, None))
            return None
        c = ctypes.c_int64()
        check(self.lib.pico_shard_apply(self.h, triples.data_ptr() if total else None, total, ctypes.byref(c)))
        return c.value

    def result(self):
        import torch
        out = torch.empty(max(self.nloc, 1), dtype=torch.int32, device=self.dev)
        check(self.lib.pico_shard_result(self.h, out.data_ptr()))
        return out[:self.nloc]

    def close(self):
        if self.h:
            check(self.lib.pico_shard_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class ShardRun:
    core_local: object
    rounds: int = 0
    frontier_sizes: list = field(default_factory=list)
    triples_exchanged: int = 0


def run_shard(shard, exchange, device) -> ShardRun:
    """The sharded HistoCore round loop for one rank.

    shard: DeviceShard (or any object with degrees/init/pack/apply/result);
    exchange: TorchDistExchange (or any object with allgather_counts /
    allgatherv).  Returns this rank's coreness and the global |C_t| sequence
    (|C_t| = |F_t|, Theorem 2), whose length is l2."""
    deg_local = shard.degrees()
    counts = exchange.allgather_counts(int(deg_local.numel()), device)
    deg_global = exchange.allgatherv(deg_local, counts)
    shard.init(deg_global)
    run = ShardRun(core_local=None)
    while True:
        trip, cnt = shard.pack()
        counts = exchange.allgather_counts(cnt, device)
        total = sum(counts)
        if total == 0:  # global convergence: no estimate changed anywhere
            break
        run.rounds += 1
        run.frontier_sizes.append(total)
        run.triples_exchanged += total
        allt = exchange.allgatherv(trip, [3 * c for c in counts])
        shard.apply(allt, total)
    run.core_local = shard.result()
    return run


def coreness_sharded(rowptr, colidx, group=None, flags: int = 0) -> ShardRun:
    """Sharded HistoCore of the full graph (rowptr/colidx on this rank's GPU;
    only this rank's rows are used): one process per GPU, torch.distributed
    group.  Returns this rank's ShardRun (core_local of its vertex range)."""
    ex = TorchDistExchange(group)
    bounds = partition(rowptr, ex.world)
    vb, ve = bounds[ex.rank], bounds[ex.rank + 1]
    rp_l, ci_l = local_rows(rowptr, colidx, vb, ve)
    shard = DeviceShard(rp_l, ci_l, vb, rowptr.numel() - 1, flags)
    try:
        run = run_shard(shard, ex, rowptr.device)
    finally:
        shard.close()
    run.v_begin, run.v_end = vb, ve
    return run


# ---------------------------------------------------------------------------
# sharded PeelOne (pico_peel_shard_*)
# ---------------------------------------------------------------------------
INT32_MAX = 2**31 - 1


class DevicePeelShard:
    """The rank's PeelOne state in libpico (owned rows [vb, vb + nloc))."""

    def __init__(self, rowptr_local, colidx_local, vb: int, n_global: int, flags: int = 0, stream=None):
        import torch
        self.lib = load()
        self.dev = rowptr_local.device
        self.rp, self.ci = rowptr_local, colidx_local
        self.nloc = rowptr_local.numel() - 1
        self.stream = stream or torch.cuda.current_stream(self.dev)
        h, km = ctypes.c_void_p(), ctypes.c_int32()
        check(self.lib.pico_peel_shard_create(self.rp.data_ptr(), self.ci.data_ptr() if self.ci.numel() else None,
                                              self.nloc, vb, n_global, flags,
                                              ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(h),
                                              ctypes.byref(km)))
        self.h, self.kmin0 = h, km.value
        self.front = torch.empty(max(self.nloc, 1), dtype=torch.int32, device=self.dev)

    def scan(self, k: int):
        c, km = ctypes.c_int64(), ctypes.c_int32()
        check(self.lib.pico_peel_shard_scan(self.h, k, self.front.data_ptr(), self.front.numel(), ctypes.byref(c),
                                            ctypes.byref(km)))
        return self.front, c.value, km.value

    def apply(self, frontier_all, total: int):
        c, km = ctypes.c_int64(), ctypes.c_int32()
        check(self.lib.pico_peel_shard_apply(self.h, frontier_all.data_ptr() if total else None, total,
                                             self.front.data_ptr(), self.front.numel(), ctypes.byref(c),
                                             ctypes.byref(km)))
        return self.front, c.value, km.value

    def result(self):
        import torch
        out = torch.empty(max(self.nloc, 1), dtype=torch.int32, device=self.dev)
        check(self.lib.pico_peel_shard_result(self.h, out.data_ptr()))
        return out[:self.nloc]

    def close(self):
        if self.h:
            check(self.lib.pico_peel_shard_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class PeelRun:
    core_local: object
    levels: int = 0
    subrounds: int = 0
    kmax: int = 0
    level_sizes: list = field(default_factory=list)  # vertices processed per non-empty level


def run_peel_shard(shard, exchange, device) -> PeelRun:
    """The sharded PeelOne loop for one rank (pico_peel_shard_* protocol).

    shard: DevicePeelShard (or any object with kmin0 / scan / apply / result);
    exchange: TorchDistExchange (or any object with allgather_pairs /
    allgatherv).  Per sub-round: an all-gather of (|F|, kmin) -- a global
    |F| of 0 ends the level, and the minimum kmin is the next level's bound --
    and an all-gatherv of F."""
    run = PeelRun(core_local=None)
    kmin = min(b for _, b in exchange.allgather_pairs(0, shard.kmin0, device))
    k = 0
    while kmin != INT32_MAX:
        k = max(k + 1, kmin)
        front, cnt, km = shard.scan(k)
        processed = 0
        while True:
            pairs = exchange.allgather_pairs(cnt, km, device)
            counts = [c for c, _ in pairs]
            kmin = min(b for _, b in pairs)
            total = sum(counts)
            if total == 0:
                break
            processed += total
            run.subrounds += 1
            allf = exchange.allgatherv(front, counts)
            front, cnt, km = shard.apply(allf, total)
        if processed:
            run.levels += 1
            run.kmax = k
            run.level_sizes.append(processed)
    run.core_local = shard.result()
    return run


def coreness_sharded_peel(rowptr, colidx, group=None, flags: int = 0) -> PeelRun:
    """Sharded PeelOne of the full graph over a torch.distributed group (one
    process per GPU; only this rank's rows are used)."""
    ex = TorchDistExchange(group)
    bounds = partition(rowptr, ex.world)
    vb, ve = bounds[ex.rank], bounds[ex.rank + 1]
    rp_l, ci_l = local_rows(rowptr, colidx, vb, ve)
    shard = DevicePeelShard(rp_l, ci_l, vb, rowptr.numel() - 1, flags)
    try:
        run = run_peel_shard(shard, ex, rowptr.device)
    finally:
        shard.close()
    run.v_begin, run.v_end = vb, ve
    return run


def coreness_loopback_peel(rowptr, colidx, nparts: int, flags: int = 0) -> PeelRun:
    """Sharded PeelOne with P logical shards on one GPU; the all-gathers are
    device concatenations.  Returns a PeelRun over all vertices."""
    import torch
    n = rowptr.numel() - 1
    bounds = partition(rowptr, nparts)
    shards = []
    run = PeelRun(core_local=None)
    try:
        for r in range(nparts):
            rp_l, ci_l = local_rows(rowptr, colidx, bounds[r], bounds[r + 1])
            shards.append(DevicePeelShard(rp_l, ci_l, bounds[r], n, flags))
        kmin = min(s.kmin0 for s in shards)
        k = 0
        while kmin != INT32_MAX:
            k = max(k + 1, kmin)
            outs = [s.scan(k) for s in shards]
            processed = 0
            while True:
                kmin = min(km for _, _, km in outs)
                total = sum(c for _, c, _ in outs)
                if total == 0:
                    break
                processed += total
                run.subrounds += 1
                allf = torch.cat([f[:c] for f, c, _ in outs])
                outs = [s.apply(allf, total) for s in shards]
            if processed:
                run.levels += 1
                run.kmax = k
                run.level_sizes.append(processed)
        run.core_local = torch.cat([s.result() for s in shards])
    finally:
        for s in shards:
            s.close()
    return run


# ---------------------------------------------------------------------------
# one-call path: the exchange inside libpico over NCCL (pico_coreness_sharded)
# ---------------------------------------------------------------------------
class NcclComm:
    """libpico's NCCL communicator (pico_comm_t) on the current CUDA device.
    The unique id is made on rank 0 and broadcast through the given
    torch.distributed group (or pass nranks=1 for a single rank)."""

    def __init__(self, group=None, nranks: int | None = None, rank: int = 0):
        import torch
        self.lib = load()
        if nranks is None:
            import torch.distributed as dist
            nranks, rank = dist.get_world_size(group), dist.get_rank(group)
        uid = (ctypes.c_uint8 * 128)()
        if rank == 0:
            check(self.lib.pico_comm_unique_id(uid))
        if nranks > 1:
            import torch.distributed as dist
            t = torch.tensor(list(bytes(uid)), dtype=torch.uint8)
            if dist.get_backend(group) == "nccl":
                t = t.cuda()
            dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
            uid = (ctypes.c_uint8 * 128)(*t.cpu().tolist())
        h = ctypes.c_void_p()
        check(self.lib.pico_comm_init(nranks, rank, uid, ctypes.byref(h)))
        self.h, self.nranks, self.rank = h, nranks, rank

    def close(self):
        if self.h:
            check(self.lib.pico_comm_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def coreness_sharded_nccl(rowptr_local, colidx_local, n_global: int, m_global: int, v_begin: int,
                          comm: NcclComm, flags: int = 0, algo: int = 0, stream=None, frontier_cap: int = 1 << 16):
    """Sharded HistoCore (algo 0) or PeelOne (algo 1) of this rank's rows
    [v_begin, v_begin + nloc) in ONE library call (pico_coreness_sharded_ex):
    the exchange runs over NCCL inside libpico.  Returns a ShardRun (core_local,
    rounds, global |C_t|; for PeelOne rounds = sub-rounds, frontier_sizes = the
    vertices processed per non-empty level, plus .levels and .kmax)."""
    import torch
    from ._lib import Stats
    lib = load()
    dev = rowptr_local.device
    nloc = rowptr_local.numel() - 1
    stream = stream or torch.cuda.current_stream(dev)
    out = torch.empty(max(nloc, 1), dtype=torch.int32, device=dev)
    st = Stats()
    fs = np.zeros(frontier_cap, dtype=np.int64)
    st.frontier_sizes = fs.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
    st.frontier_sizes_cap = frontier_cap
    check(lib.pico_coreness_sharded_ex(comm.h, rowptr_local.data_ptr(),
                                       colidx_local.data_ptr() if colidx_local.numel() else None, n_global, m_global,
                                       v_begin, v_begin + nloc, algo, out.data_ptr() if nloc else None,
                                       ctypes.c_void_p(stream.cuda_stream), flags, ctypes.byref(st)))
    if algo == 1:
        run = ShardRun(core_local=out[:nloc], rounds=int(st.subrounds))
        run.levels, run.kmax = int(st.levels), int(st.kmax)
        run.frontier_sizes = [int(x) for x in fs[:run.levels]]
        return run
    run = ShardRun(core_local=out[:nloc], rounds=int(st.rounds))
    run.frontier_sizes = [int(x) for x in fs[:run.rounds]]
    return run


# ---------------------------------------------------------------------------
# loopback: P logical shards on one GPU (parity of the sharded kernels)
# ---------------------------------------------------------------------------
def coreness_loopback(rowptr, colidx, nparts: int, flags: int = 0):
    """P shards in one process; the exchange is a device concatenation.
    Returns (coreness of all vertices, rounds l2, [|C_t|])."""
    import torch
    n = rowptr.numel() - 1
    bounds = partition(rowptr, nparts)
    shards = []
    try:
        for r in range(nparts):
            rp_l, ci_l = local_rows(rowptr, colidx, bounds[r], bounds[r + 1])
            shards.append(DeviceShard(rp_l, ci_l, bounds[r], n, flags))
        deg = torch.cat([s.degrees() for s in shards])
        for s in shards:
            s.init(deg)
        sizes = []
        while True:
            packs = [s.pack() for s in shards]
            total = sum(c for _, c in packs)
            if total == 0:
                break
            sizes.append(total)
            allt = torch.cat([t[:3 * c] for t, c in packs])
            for s in shards:
                s.apply(allt, total)
        core = torch.cat([s.result() for s in shards])
    finally:
        for s in shards:
            s.close()
    return core, len(sizes), sizes
