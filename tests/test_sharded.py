"""T7: sharded HistoCore.

CPU: the partition, and the exchange / round protocol of
paper_2402_15253_b200.sharded.run_shard over a real torch.distributed gloo
group of world size 2.  The shard compute there is a test-only mock: the plain
synchronous Index2core iteration (Alg 2) on the rank's owned
vertices, whose changed sets are exactly HistoCore's C_t.

GPU: the real shard kernels (include/pico_shard.h) in loopback mode -- P
logical shards on one GPU, exchange = device concatenation -- against the
oracle (coreness bit-exact, l2 and every |C_t| equal to the Jacobi sweeps)."""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2402_15253_b200 import sharded


# ---------------------------------------------------------------- partition
@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8])
def test_partition_arc_balanced(parts):
    rp, ci = synth.to_numpy(*synth.CONFIGS["R14"].build())
    b = sharded.partition(rp, parts)
    assert b[0] == 0 and b[-1] == rp.size - 1 and len(b) == parts + 1
    assert all(x <= y for x, y in zip(b, b[1:]))
    arcs = int(rp[-1])
    dmax = int(np.diff(rp).max())
    for r in range(parts):
        got = int(rp[b[r + 1]] - rp[b[r]])
        assert abs(got - arcs / parts) <= dmax + 1  # balanced up to one row


def test_partition_degenerate():
    rp = np.array([0, 0, 0, 2, 2, 4], dtype=np.int64)  # isolated + small rows
    b = sharded.partition(rp, 4)
    assert b[0] == 0 and b[-1] == 5 and sorted(b) == b


def test_local_rows_slices():
    rp, ci = synth.CONFIGS["R12"].build()
    b = sharded.partition(rp, 3)
    total = 0
    for r in range(3):
        rl, cl = sharded.local_rows(rp, ci, b[r], b[r + 1])
        assert int(rl[0]) == 0 and int(rl[-1]) == cl.numel()
        total += cl.numel()
    assert total == ci.numel()


@pytest.mark.parametrize("cfg", ["R12", "C1"])
def test_rows_generation_matches_slices(cfg):
    """Per-rank generation (synth rmat_rows, used by the sharded bench so that
    C5 = RMAT-30 never exists whole on one GPU) gives exactly the rows of the
    full graph: equal vertex ranges at P = 1, 3, 4."""
    c = synth.CONFIGS[cfg]
    rp, ci = c.build()
    n = rp.numel() - 1
    for parts in (1, 3, 4):
        b = sharded.partition_vertices(n, parts)
        for r in range(parts):
            rl, cl = c.build_rows(b[r], b[r + 1])
            el, ecl = sharded.local_rows(rp, ci, b[r], b[r + 1])
            assert torch.equal(rl, el) and torch.equal(cl, ecl), (cfg, parts, r)
    with pytest.raises(ValueError):
        synth.CONFIGS["C2"].build_rows(0, 10)  # compacted configs renumber globally


# ------------------------------------------------- mock shard (test only)
class JacobiShard:
    """Owned vertices [vb, ve): synchronous Index2core on a replica of every
    neighbour's estimate, updated only from exchanged triples."""

    def __init__(self, rp_l, ci_l, vb, n_global):
        self.rp, self.ci = rp_l, ci_l
        self.vb, self.nloc = vb, rp_l.size - 1
        self.pending = []

    def degrees(self):
        return torch.from_numpy(np.diff(self.rp).astype(np.int32))

    def init(self, deg_global):
        self.rep = deg_global.numpy().astype(np.int64).copy()
        self.val = np.diff(self.rp).astype(np.int64)
        self._sweep()

    def _sweep(self):
        new = np.array([oracle.hindex(self.rep[self.ci[self.rp[v]:self.rp[v + 1]]])
                        for v in range(self.nloc)], dtype=np.int64)
        ch = np.flatnonzero(new != self.val)
        self.pending = [(self.vb + v, int(self.val[v]), int(new[v])) for v in ch]
        self.val = new

    def pack(self):
        flat = np.array(self.pending, dtype=np.int32).reshape(-1)
        return torch.from_numpy(flat if flat.size else np.zeros(3, np.int32)), len(self.pending)

    def apply(self, triples, total):
        t = triples.numpy().reshape(-1, 3)
        for v, old, new in t:
            assert self.rep[v] == old
            self.rep[v] = new
        self._sweep()
        return len(self.pending)

    def result(self):
        return torch.from_numpy(self.val.astype(np.int32))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, cfg, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rp, ci = synth.CONFIGS[cfg].build() if cfg in synth.CONFIGS else synth.g1()
        rpn, cin = synth.to_numpy(rp, ci)
        ex = sharded.TorchDistExchange()
        b = sharded.partition(rpn, world)
        rl, cl = sharded.local_rows(rp, ci, b[rank], b[rank + 1])
        shard = JacobiShard(rl.numpy(), cl.numpy(), b[rank], rpn.size - 1)
        run = sharded.run_shard(shard, ex, torch.device("cpu"))
        counts = ex.allgather_counts(run.core_local.numel(), torch.device("cpu"))
        core = ex.allgatherv(run.core_local, counts)
        if rank == 0:
            out.put((core.numpy().tolist(), run.rounds, run.frontier_sizes))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", ["G1", "R12"])
def test_gloo_world2_protocol(cfg):
    """world_size 2 over gloo: the sharded round protocol (count all-gather =
    convergence test, triple all-gatherv, rank-ordered degree exchange) yields
    the oracle coreness, l2 and |C_t| sequence."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, cfg, q)) for r in range(2)]
    for p in procs:
        p.start()
    core, rounds, sizes = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rp, ci = synth.to_numpy(*(synth.CONFIGS[cfg].build() if cfg in synth.CONFIGS else synth.g1()))
    assert core == oracle.bz(rp, ci).tolist()
    _, l2, fs = oracle.jacobi_rounds(rp, ci)
    assert rounds == l2 and sizes == fs


class NumpyPeelShard:
    """Owned vertices [vb, ve): the level-synchronous peel on owned residual
    degrees, decremented only through exchanged frontier vertices (the
    pico_peel_shard_* protocol on the host)."""

    def __init__(self, rp_l, ci_l, vb, n_global):
        self.vb, self.nloc = vb, rp_l.size - 1
        self.core = np.diff(rp_l).astype(np.int64)
        self.csc = {}
        for u in range(self.nloc):
            for v in ci_l[rp_l[u]:rp_l[u + 1]]:
                self.csc.setdefault(int(v), []).append(u)
        alive = self.core[self.core > 0]
        self.kmin0 = int(alive.min()) if alive.size else sharded.INT32_MAX
        self.k = 0
        self.bound = sharded.INT32_MAX

    def scan(self, k):
        self.k = k
        keep = self.core > k
        self.bound = int(self.core[keep].min()) if keep.any() else sharded.INT32_MAX
        f = np.flatnonzero(self.core == k) + self.vb
        return torch.from_numpy(f.astype(np.int32)), f.size, self.bound

    def apply(self, allf, total):
        k, nxt = self.k, []
        for v in allf.numpy()[:total]:
            for u in self.csc.get(int(v), []):
                if self.core[u] > k:  # guard, then the clamped decrement
                    self.core[u] -= 1
                    if self.core[u] == k:
                        nxt.append(u + self.vb)
                    else:
                        self.bound = min(self.bound, int(self.core[u]))
        f = np.array(nxt, dtype=np.int32)
        return torch.from_numpy(f), f.size, self.bound

    def result(self):
        return torch.from_numpy(self.core.astype(np.int32))


def _gloo_peel_worker(rank, world, port, cfg, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rp, ci = synth.CONFIGS[cfg].build() if cfg in synth.CONFIGS else synth.g1()
        rpn, cin = synth.to_numpy(rp, ci)
        ex = sharded.TorchDistExchange()
        b = sharded.partition(rpn, world)
        rl, cl = sharded.local_rows(rp, ci, b[rank], b[rank + 1])
        shard = NumpyPeelShard(rl.numpy(), cl.numpy(), b[rank], rpn.size - 1)
        run = sharded.run_peel_shard(shard, ex, torch.device("cpu"))
        counts = ex.allgather_counts(run.core_local.numel(), torch.device("cpu"))
        core = ex.allgatherv(run.core_local, counts)
        if rank == 0:
            out.put((core.numpy().tolist(), run.levels, run.subrounds, run.kmax, run.level_sizes))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", ["G1", "R12"])
def test_gloo_world2_peel_protocol(cfg):
    """world_size 2 over gloo: the sharded PeelOne protocol ((|F|, kmin)
    all-gather = level test and next-level bound, F all-gatherv) yields the
    oracle coreness and the level-synchronous reference's level / sub-round
    counts."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_peel_worker, args=(r, 2, port, cfg, q)) for r in range(2)]
    for p in procs:
        p.start()
    core, levels, subrounds, kmax, sizes = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rp, ci = synth.to_numpy(*(synth.CONFIGS[cfg].build() if cfg in synth.CONFIGS else synth.g1()))
    ref = oracle.bz(rp, ci)
    assert core == ref.tolist()
    _, km, lv, sr = oracle.peel_levels(rp, ci)
    assert (levels, subrounds, kmax) == (lv, sr, km)
    nz = ref[ref > 0]
    assert sizes == [int((nz == c).sum()) for c in np.unique(nz)]


def test_shard_capi_argument_errors():
    import ctypes
    import paper_2402_15253_b200 as pico
    from paper_2402_15253_b200 import build
    build.build()
    lib = pico.load()
    h = ctypes.c_void_p()
    rp = np.zeros(3, dtype=np.int64)
    # range beyond n_global / negative / NULL out
    assert lib.pico_shard_create(rp.ctypes.data, None, 2, 5, 4, 0, None, ctypes.byref(h)) == 1
    assert lib.pico_shard_create(rp.ctypes.data, None, -1, 0, 4, 0, None, ctypes.byref(h)) == 1
    assert lib.pico_shard_create(rp.ctypes.data, None, 2, 0, 4, 0, None, None) == 1
    assert lib.pico_shard_destroy(None) == 0
    km = ctypes.c_int32()
    assert lib.pico_peel_shard_create(rp.ctypes.data, None, 2, 5, 4, 0, None, ctypes.byref(h), ctypes.byref(km)) == 1
    assert lib.pico_peel_shard_create(rp.ctypes.data, None, 2, 0, 4, 0, None, None, ctypes.byref(km)) == 1
    assert lib.pico_peel_shard_scan(None, 1, None, 0, None, None) == 1
    assert lib.pico_peel_shard_destroy(None) == 0


# ---------------------------------------------------------------- GPU
def _graphs():
    from conftest import csr_np, parse_g1
    g = parse_g1()
    edges = [tuple(int(x) for x in p.split("-")) for p in g["edges"].split()]
    out = [("G1", csr_np(6, edges)),
           ("K20", csr_np(20, [(i, j) for i in range(20) for j in range(i + 1, 20)])),
           ("star", csr_np(101, [(0, i) for i in range(1, 101)]))]
    for i, (n, p) in enumerate([(150, 0.05), (200, 0.2)]):
        out.append((f"er{i}", synth.to_numpy(*synth.erdos_renyi(n, p, seed=3000 + i))))
    out.append(("cl", synth.to_numpy(*synth.chung_lu(3000, 10.0, 2.2, seed=3100))))
    out.append(("R12", synth.to_numpy(*synth.CONFIGS["R12"].build())))
    out.append(("R14", synth.to_numpy(*synth.CONFIGS["R14"].build())))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8])
def test_loopback_parity(parts):
    import paper_2402_15253_b200 as pico
    dev = torch.device("cuda:0")
    for name, (rp, ci) in _graphs():
        ref = oracle.bz(rp, ci)
        _, l2, fs = oracle.jacobi_rounds(rp, ci)
        for fl in (0, pico.F_TINY_TILES, pico.F_PULL_ALWAYS, pico.F_PULL_ALWAYS | pico.F_TINY_TILES):
            core, rounds, sizes = sharded.coreness_loopback(torch.from_numpy(rp).to(dev),
                                                            torch.from_numpy(ci).to(dev), parts, fl)
            got = core.cpu().numpy()
            assert np.array_equal(got, ref), (name, parts, fl, np.flatnonzero(got != ref)[:5])
            assert rounds == l2 and sizes == fs, (name, parts, fl)


@pytest.mark.gpu
def test_loopback_c1():
    rp, ci = synth.to_numpy(*synth.CONFIGS["C1"].build())
    dev = torch.device("cuda:0")
    ref = oracle.bz(rp, ci)
    _, l2, fs = oracle.jacobi_rounds(rp, ci)
    import paper_2402_15253_b200 as pico
    for parts in (2, 8):
        for fl in (0, pico.F_PULL_ALWAYS):  # push rounds over the CSC / pull rounds over the edge list
            core, rounds, sizes = sharded.coreness_loopback(torch.from_numpy(rp).to(dev),
                                                            torch.from_numpy(ci).to(dev), parts, fl)
            assert np.array_equal(core.cpu().numpy(), ref) and rounds == l2 and sizes == fs


@pytest.mark.gpu
@pytest.mark.parametrize("parts", [1, 2, 3, 8])
def test_loopback_peel_parity(parts):
    """Sharded PeelOne (P logical shards, device concatenation as the
    exchange): bit-exact coreness, and the non-empty levels, BSP sub-rounds,
    k_max and per-level sizes of the single-GPU PeelOne / level-synchronous
    reference, for every P."""
    import paper_2402_15253_b200 as pico
    dev = torch.device("cuda:0")
    for name, (rp, ci) in _graphs():
        ref = oracle.bz(rp, ci)
        _, km, lv, sr = oracle.peel_levels(rp, ci)
        nz = ref[ref > 0]
        per_level = [int((nz == c).sum()) for c in np.unique(nz)]
        for fl in (0, pico.F_TINY_TILES, pico.F_CLAMP_CAS | pico.F_STATS):
            run = sharded.coreness_loopback_peel(torch.from_numpy(rp).to(dev), torch.from_numpy(ci).to(dev),
                                                 parts, fl)
            got = run.core_local.cpu().numpy()
            assert np.array_equal(got, ref), (name, parts, fl, np.flatnonzero(got != ref)[:5])
            assert (run.levels, run.subrounds, run.kmax) == (lv, sr, km), (name, parts, fl)
            assert run.level_sizes == per_level


@pytest.mark.gpu
def test_peel_shard_step_checks():
    """pico_peel_shard_*: a frontier buffer shorter than nloc, k < 1 and a
    negative total are PICO_EINVAL; an isolated-only shard reports INT32_MAX."""
    import paper_2402_15253_b200 as pico
    dev = torch.device("cuda:0")
    rp, ci = synth.to_numpy(*synth.CONFIGS["R12"].build())
    rp_t, ci_t = torch.from_numpy(rp).to(dev), torch.from_numpy(ci).to(dev)
    lib = pico.load()
    n = rp.size - 1
    sh = sharded.DevicePeelShard(rp_t, ci_t, 0, n)
    try:
        c, km = ctypes.c_int64(), ctypes.c_int32()
        small = torch.empty(n - 1, dtype=torch.int32, device=dev)
        assert lib.pico_peel_shard_scan(sh.h, 1, small.data_ptr(), n - 1, ctypes.byref(c), ctypes.byref(km)) == 1
        assert lib.pico_peel_shard_scan(sh.h, 0, sh.front.data_ptr(), n, ctypes.byref(c), ctypes.byref(km)) == 1
        assert lib.pico_peel_shard_apply(sh.h, None, -1, sh.front.data_ptr(), n, ctypes.byref(c),
                                         ctypes.byref(km)) == 1
        assert sh.kmin0 == int(np.diff(rp)[np.diff(rp) > 0].min())
    finally:
        sh.close()
    iso = torch.zeros(4, dtype=torch.int64, device=dev)  # three isolated vertices
    sh = sharded.DevicePeelShard(iso, torch.empty(0, dtype=torch.int32, device=dev), 0, 3)
    try:
        assert sh.kmin0 == sharded.INT32_MAX
        assert sh.result().tolist() == [0, 0, 0]
    finally:
        sh.close()


@pytest.mark.gpu
def test_loopback_peel_c1():
    rp, ci = synth.to_numpy(*synth.CONFIGS["C1"].build())
    dev = torch.device("cuda:0")
    ref = oracle.bz(rp, ci)
    _, km, lv, sr = oracle.peel_levels(rp, ci)
    for parts in (2, 8):
        run = sharded.coreness_loopback_peel(torch.from_numpy(rp).to(dev), torch.from_numpy(ci).to(dev), parts)
        assert np.array_equal(run.core_local.cpu().numpy(), ref)
        assert (run.levels, run.subrounds, run.kmax) == (lv, sr, km)


# ------------------------------------------------ one-call NCCL path (C ABI)
@pytest.mark.gpu
def test_sharded_abi_single_rank_nccl():
    """pico_coreness_sharded_ex with the exchange inside libpico over NCCL, one
    rank: bit-exact coreness and the Jacobi |F_t| sequence; argument checks."""
    import torch
    import oracle
    import paper_2402_15253_b200 as pico
    from paper_2402_15253_b200 import sharded
    dev = torch.device("cuda:0")
    rp_np, ci_np = synth.to_numpy(*synth.CONFIGS["R12"].build())
    ref = oracle.bz(rp_np, ci_np)
    _, l2, sizes = oracle.jacobi_rounds(rp_np, ci_np)
    rp, ci = torch.from_numpy(rp_np).to(dev), torch.from_numpy(ci_np).to(dev)
    n, m = rp.numel() - 1, ci.numel() // 2
    comm = sharded.NcclComm(nranks=1, rank=0)
    try:
        for fl in (0, pico.F_TINY_TILES, pico.F_PULL_ALWAYS, pico.F_PULL_ALWAYS | pico.F_TINY_TILES):
            run = sharded.coreness_sharded_nccl(rp, ci, n, m, 0, comm, flags=fl)
            torch.cuda.synchronize()
            assert np.array_equal(run.core_local.cpu().numpy(), ref)
            assert run.rounds == l2 and run.frontier_sizes == sizes
        lib = pico.load()
        out = torch.empty(n, dtype=torch.int32, device=dev)
        s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        # ranges must tile [0, n_global); arcs must sum to 2m; only HistoCore / PeelOne shard
        assert lib.pico_coreness_sharded(comm.h, rp.data_ptr(), ci.data_ptr(), n + 5, m, 0, n, 0,
                                         out.data_ptr(), s) == 1
        assert lib.pico_coreness_sharded(comm.h, rp.data_ptr(), ci.data_ptr(), n, m + 1, 0, n, 0,
                                         out.data_ptr(), s) == 1
        assert lib.pico_coreness_sharded(comm.h, rp.data_ptr(), ci.data_ptr(), n, m, 0, n, 3,
                                         out.data_ptr(), s) == 1
        # sharded PeelOne through the same entry point
        _, km, lv, sr = oracle.peel_levels(rp_np, ci_np)
        for fl in (0, pico.F_TINY_TILES):
            run = sharded.coreness_sharded_nccl(rp, ci, n, m, 0, comm, flags=fl, algo=1)
            torch.cuda.synchronize()
            assert np.array_equal(run.core_local.cpu().numpy(), ref)
            assert (run.levels, run.rounds, run.kmax) == (lv, sr, km)
    finally:
        comm.close()


@pytest.mark.gpu
@pytest.mark.parametrize("batch", ["1", "3", "4"])
def test_sharded_lsa_exchange_single_rank(batch, monkeypatch):
    """PICO_F_LSA_EXCHANGE: the round's exchange on the device over NCCL's
    device API (symmetric window, LSA barrier, peer loads), rounds enqueued in
    batches with one host read per batch.  One rank: bit-exact coreness, l2
    and every global |C_t| of the Jacobi reference, on R12 and C1, push,
    pull-always and tiny-tile schedules, batch sizes that end the run at, before
    and past a batch boundary."""
    import torch
    import oracle
    import paper_2402_15253_b200 as pico
    from paper_2402_15253_b200 import sharded
    monkeypatch.setenv("PICO_LSA_BATCH", batch)
    dev = torch.device("cuda:0")
    comm = sharded.NcclComm(nranks=1, rank=0)
    try:
        for cfg in ("R12", "C1"):
            rp_np, ci_np = synth.to_numpy(*synth.CONFIGS[cfg].build())
            ref = oracle.bz(rp_np, ci_np)
            _, l2, sizes = oracle.jacobi_rounds(rp_np, ci_np)
            rp, ci = torch.from_numpy(rp_np).to(dev), torch.from_numpy(ci_np).to(dev)
            n, m = rp.numel() - 1, ci.numel() // 2
            for fl in (0, pico.F_TINY_TILES, pico.F_PULL_ALWAYS, pico.F_PULL_ALWAYS | pico.F_TINY_TILES):
                run = sharded.coreness_sharded_nccl(rp, ci, n, m, 0, comm, flags=fl | pico.F_LSA_EXCHANGE)
                torch.cuda.synchronize()
                assert np.array_equal(run.core_local.cpu().numpy(), ref), (cfg, fl)
                assert run.rounds == l2 and run.frontier_sizes == sizes, (cfg, fl, run.rounds, l2)
            # sharded PeelOne, its level loop on the device (the same window, 1-word items)
            _, km, lv, sr = oracle.peel_levels(rp_np, ci_np)
            nz = ref[ref > 0]
            per_level = [int((nz == k).sum()) for k in np.unique(nz)]
            for fl in (0, pico.F_TINY_TILES, pico.F_CLAMP_CAS):
                run = sharded.coreness_sharded_nccl(rp, ci, n, m, 0, comm, flags=fl | pico.F_LSA_EXCHANGE, algo=1)
                torch.cuda.synchronize()
                assert np.array_equal(run.core_local.cpu().numpy(), ref), (cfg, "peel", fl)
                assert (run.levels, run.rounds, run.kmax) == (lv, sr, km), (cfg, fl, run.levels, run.rounds)
                assert run.frontier_sizes == per_level
    finally:
        comm.close()
