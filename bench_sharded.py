"""bench.py --gpus N (N > 1, launched by torchrun): sharded HistoCore
(SURVEY 8(e)), or sharded PeelOne with --algo peelone.  One process per GPU, NCCL over NVLink/NVSwitch for the
exchange (torch.distributed), libpico kernels for every compute step.

A step = one complete sharded coreness computation of the graph (shard
creation with the per-rank CSC build, degree exchange, init, every round's
pack / all-gatherv / apply, result).  Timed with CUDA events bracketed by a
barrier + synchronize on both sides; the step time is the MAX over ranks;
value = m / that time ("scaling": "strong": the graph is fixed as N grows).
Every rank builds the same seeded graph and uses only its own rows.
"""
from __future__ import annotations

import json
import os
import time

import numpy as np


def fixed_point_violations(rp_l, ci_l, vb: int, core, chunk: int = 1 << 27) -> int:
    """Rows of this rank whose estimate is not the h-index of its neighbours'
    (#nbrs with core >= c is >= c and #nbrs with core >= c+1 is <
    c+1), or that break 0 <= core <= deg / core = 0 iff deg = 0.
    Chunked over the rank's arcs (torch, on the rank's GPU)."""
    import torch
    nloc = rp_l.numel() - 1
    if nloc == 0:
        return 0
    deg = rp_l[1:] - rp_l[:-1]
    cv = core[vb:vb + nloc].to(torch.int64)
    bad = int(((cv < 0) | (cv > deg) | ((cv == 0) != (deg == 0))).sum().item())
    ge = torch.zeros(nloc, dtype=torch.int64, device=core.device)
    gt = torch.zeros(nloc, dtype=torch.int64, device=core.device)
    arcs = ci_l.numel()
    for a0 in range(0, arcs, chunk):
        a1 = min(arcs, a0 + chunk)
        rows = torch.searchsorted(rp_l, torch.arange(a0, a1, device=core.device, dtype=torch.int64), right=True) - 1
        cu = core[ci_l[a0:a1].to(torch.int64)].to(torch.int64)
        c = cv[rows]
        ge += torch.bincount(rows, weights=(cu >= c).to(torch.float64), minlength=nloc).to(torch.int64)
        gt += torch.bincount(rows, weights=(cu >= c + 1).to(torch.float64), minlength=nloc).to(torch.int64)
        del rows, cu, c
    live = deg > 0
    bad += int((live & ((ge < cv) | (gt >= cv + 1))).sum().item())
    return bad


def bench_sharded(args):
    import torch
    import torch.distributed as dist

    import bench
    import paper_2402_15253_b200 as pico
    from paper_2402_15253_b200 import sharded

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    # NCCL's INIT log (ranks, channels, NVLS) goes to stderr so the rank set can be
    # verified; stdout carries exactly one JSON line
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    ex = sharded.TorchDistExchange()
    stream = torch.cuda.current_stream(dev)

    import synth
    cfg = synth.CONFIGS[args.config]
    per_rank = not cfg.compact  # uncompacted recipes (T, C5, C1): each rank generates only its rows
    rp = ci = None
    t_gen = time.time()
    if per_rank:
        n = cfg.n
        bounds = sharded.partition_vertices(n, world)
        vb, ve = bounds[rank], bounds[rank + 1]
        rp_l, ci_l = cfg.build_rows(vb, ve, device=dev)
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        arcs_t = torch.tensor([ci_l.numel()], dtype=torch.int64, device=dev)
        dist.all_reduce(arcs_t)
        m = int(arcs_t.item()) // 2
        gen_note = "per rank: each GPU generated only its own rows (equal vertex ranges)"
    else:
        cfg, rp, ci = bench.build_graph(args.config, dev)
        n, m = rp.numel() - 1, ci.numel() // 2
        bounds = sharded.partition(rp, world)
        vb, ve = bounds[rank], bounds[rank + 1]
        rp_l, ci_l = sharded.local_rows(rp, ci, vb, ve)
        gen_note = "whole graph on every rank (compaction renumbers globally), arc-balanced ranges"
    t_gen = time.time() - t_gen
    if rank == 0:
        bench.log(f"[bench-sharded] {args.config}: n={n} m={m} local arcs {ci_l.numel()} generated in {t_gen:.1f}s ({gen_note})")

    comm, exchange_note = None, "torch.distributed"
    if args.exchange in ("nccl", "lsa"):
        try:
            comm = sharded.NcclComm()
            exchange_note = "NCCL inside libpico (pico_coreness_sharded)"
            if args.exchange == "lsa":
                args.flags |= pico.F_LSA_EXCHANGE
                exchange_note = ("NCCL device API inside libpico (symmetric window, LSA peer loads, one LSA "
                                 "barrier per round, no host synchronisation per round)")
        except Exception as e:  # no usable libnccl: the torch.distributed exchange (also GPU, also NCCL)
            exchange_note = f"torch.distributed (in-library NCCL unavailable: {e})"

    peel = args.algo == "peelone"

    def run_once(rp_d, ci_d):
        if comm is not None:  # one library call; the exchange runs over NCCL inside libpico
            r = sharded.coreness_sharded_nccl(rp_d, ci_d, n, m, vb, comm, flags=args.flags, algo=1 if peel else 0)
            if peel:
                r.subrounds = r.rounds
                r.exchanged = sum(r.frontier_sizes)
            else:
                r.exchanged = sum(r.frontier_sizes)
            return r
        if peel:
            shard = sharded.DevicePeelShard(rp_d, ci_d, vb, n, args.flags)
            try:
                r = sharded.run_peel_shard(shard, ex, dev)
            finally:
                shard.close()
            r.exchanged = sum(r.level_sizes)
            return r
        shard = sharded.DeviceShard(rp_d, ci_d, vb, n, args.flags)
        try:
            r = sharded.run_shard(shard, ex, dev)
        finally:
            shard.close()
        r.exchanged = r.triples_exchanged
        return r

    def step():
        return run_once(rp_l, ci_l)

    for w in range(args.warmup):
        try:
            run = step()
        except Exception as e:
            if comm is None or w > 0:
                raise
            # the in-library exchange failed on this box: every rank falls back together
            comm.close()
            comm = None
            exchange_note = f"torch.distributed (in-library NCCL failed: {e})"
            run = step()
    dist.barrier()
    torch.cuda.synchronize()
    clk = bench.ClockSampler(local) if rank == 0 else None
    if clk:
        clk.__enter__()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        run = step()
    e1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    if clk:
        clk.__exit__(None, None, None)
    ms_rank = e0.elapsed_time(e1) / args.steps
    ms = ex.max_over_ranks(ms_rank, dev)

    # parity: the assembled coreness against the single-GPU path (itself
    # bit-exact vs the oracle in tests and in the N=1 bench) on rank 0, where
    # the whole graph fits one GPU; always, on every rank, the h-index fixed
    # point of its own rows against the assembled vector
    counts = ex.allgather_counts(run.core_local.numel(), dev)
    core = ex.allgatherv(run.core_local, counts)
    fp_bad = fixed_point_violations(rp_l, ci_l, vb, core)
    fp_bad = int(ex.max_over_ranks(float(fp_bad), dev))
    parity = f"h-index fixed point on every rank's rows: {'ok' if fp_bad == 0 else f'{fp_bad} violations'}"
    ref_stats = None
    if rank == 0 and n <= (1 << 27):
        if rp is None:
            rp, ci = cfg.build(device=dev)
        ref_stats = pico.Stats()
        ref_fs = np.zeros(1 << 16, dtype=np.int64)
        ref_ra = np.zeros(1 << 16, dtype=np.int64)
        ref = pico.coreness(rp, ci, flags=pico.F_STATS, stats=ref_stats, frontier_sizes=ref_fs, round_arcs=ref_ra)
        parity = ("bit-exact vs single-GPU" if torch.equal(core, ref) else "MISMATCH vs single-GPU") + "; " + parity
        if not args.no_oracle and n * 1 <= (8 << 20):
            import oracle
            r_np, c_np = synth.to_numpy(rp, ci)
            if np.array_equal(oracle.bz(r_np, c_np), core.cpu().numpy()):
                parity = "bit-exact vs oracle; " + parity
            else:
                parity = "MISMATCH vs oracle; " + parity
        del rp, ci
        torch.cuda.empty_cache()

    # e2e: local rows from pinned host memory -> device, sharded run, result
    # back to pinned host memory, per step
    rp_h = rp_l.cpu().pin_memory()
    ci_h = ci_l.cpu().pin_memory()
    out_h = torch.empty(max(rp_l.numel() - 1, 1), dtype=torch.int32).pin_memory()
    e2e_steps = max(3, min(args.steps, 5))
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        rp_d = rp_h.to(dev, non_blocking=True)
        ci_d = ci_h.to(dev, non_blocking=True)
        r2 = run_once(rp_d, ci_d)
        out_h[:r2.core_local.numel()].copy_(r2.core_local, non_blocking=True)
        torch.cuda.synchronize()
    dist.barrier()
    e2e_t = ex.max_over_ranks((time.perf_counter() - t0) / e2e_steps, dev)

    if rank == 0:
        peak, src = bench.hbm_peak()
        # roofline: the method's bytes of the whole graph (identical rounds and
        # frontiers at every P; counted by a single-GPU STATS run where the
        # graph fits one GPU) over the max-over-ranks step time and N peaks
        roof = {"bound": "hbm", "achieved": None, "peak": peak * world, "unit": "GB/s", "frac": None,
                "traffic": None, "peak_source": src + f" x {world} GPUs", "kernel": "whole sharded step"}
        if ref_stats is not None and not peel:
            sd = ref_stats.to_dict()
            b = bench.hc_bytes(n, m, sd, int(ref_fs[0]), int(ref_ra[:sd["rounds"]].sum()))
            tot = sum(b.values())
            roof.update({"achieved": tot / (ms * 1e-3) / 1e9, "frac": tot / (ms * 1e-3) / 1e9 / (peak * world),
                         "alg_bytes": b})
        else:
            roof["note"] = "method bytes need a single-GPU STATS run, which does not fit one GPU here"
        # cpu_baseline: the oracle on this host, one core, on the reference
        # arm's bounded sample of the workload
        cpu_base = None
        if not args.no_oracle:
            import oracle
            _, rp_s, ci_s, what = bench.reference_graph(args.config, dev)
            r_np, c_np = synth.to_numpy(rp_s, ci_s)
            del rp_s, ci_s
            _, times = bench.oracle_baseline(r_np, c_np, budget_s=10.0, max_runs=3)
            tb = min(times)
            cpu_base = {"value": (c_np.size // 2) / tb, "unit": bench.UNIT, "cores": 1, "kind": "oracle",
                        "sample": f"{what} (n={r_np.size - 1}, m={c_np.size // 2}), serial BZ, best of {len(times)}",
                        "ms": 1e3 * tb}
        launches = (8 + 3 * run.subrounds + 3 * run.levels) if peel else 12 + 4 * run.rounds
        if peel:
            iters = {"peelone_levels": run.levels, "peelone_subrounds": run.subrounds, "kmax": run.kmax}
            exch = {"frontier_ids_per_step": run.exchanged, "bytes_per_rank_per_step": 4 * run.exchanged,
                    "collectives_per_step": run.subrounds + run.levels + 1, "partition": bounds}
            par = (f"1-D vertex partition x{world} (per sub-round: all-gather of (|F|, kmin) and allgatherv of "
                   "the frontier over NCCL: " + exchange_note + ")")
        else:
            iters = {"histocore_l2": run.rounds}
            exch = {"triples_per_step": run.exchanged, "bytes_per_rank_per_step": 12 * run.exchanged,
                    "partition": bounds}
            par = f"1-D vertex partition x{world} (allgatherv of changed triples over NCCL: " + exchange_note + ")"
        out = {
            "metric": bench.METRIC, "value": m / (ms * 1e-3), "unit": bench.UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": cfg.note, "config": args.config, "algo": f"{args.algo}-sharded", "n": n, "m": m,
                       "parallelism": par, "generation": gen_note,
                       "l2_flush": "inputs larger than L2"},
            "roofline": roof,
            "cpu_baseline": cpu_base,
            "e2e": {"value": m / e2e_t, "unit": bench.UNIT, "ms_per_step": 1e3 * e2e_t,
                    "h2d_bytes_per_step": int(8 * n + 4 * 2 * m), "d2h_bytes_per_step": int(4 * n)},
            "gpu_launches": launches * args.steps * world,
            "clocks": clk.summary() if clk else None,
            "parity": parity,
            "iterations": iters,
            "exchange": exch,
        }
        print(json.dumps(out), flush=True)
    dist.barrier()
    if comm is not None:
        comm.close()
    dist.destroy_process_group()
    return 0
