#!/usr/bin/env python
"""bench.py -- k-core decomposition throughput on B200 (BASELINE.json metric:
"k-core decomposition edges/sec and ms (1/2/4/8 B200), % of HBM roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2]
                    [--algo histocore|peelone] [--impl pico|reference]

A step = one coreness computation of the whole graph through the C ABI
(pico_coreness_ex: device-resident CSR in, device-resident coreness out,
workspace allocation included).  value = undirected edges m
/ step time (edges/s).  Inputs (colidx 4*2m bytes, histogram 4*2m bytes) are
larger than the 126 MB L2, so no explicit flush is needed between steps.

N = 1: the HistoCore primary kernel on configs[1] (LiveJournal-shaped); PeelOne
is measured on the same graph and reported alongside.  N > 1 (torchrun, one
process per GPU): sharded HistoCore over a 1-D vertex partition,
value = m / max-over-ranks step time, "scaling": "strong".

--impl reference: the CPU oracle (serial Batagelj-Zaversnik, oracle/) timed on
this box's host cores on the same workload -- the reference arm of this tier.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "k-core decomposition edges/sec and ms (1/2/4/8 B200), % of HBM roofline"
UNIT = "edges/s"
DEFAULT_CONFIG = "C2"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# roofline model: algorithmic bytes per kernel slot (DESIGN.md "Algorithmic
# bytes"; SURVEY 8(d) 4-byte access model, each logical access counted once)
# ---------------------------------------------------------------------------
def hc_bytes(n: int, m: int, st: dict, f1: int, relabelled: bool = False) -> dict:
    """B_alg = 8(n+1) + 4*2m [colidx] + 4*2m [gather deg] + 4*W1
    [init slots] + 12n [core/oldcore init, initial cnt] + sum_t (32|F_t| +
    4 bins_t + 8 S_t + 16 G_t), split by kernel slot: degree = rowptr + the
    two estimate arrays; init = colidx + degree gathers + W1 + core + the
    round-1 frontier (32|F_1|); rounds = the per-round terms for t >= 2 with
    S_t = arcs scanned (push: rows of C_t; pull: rows streamed) and G_t =
    guarded arcs (two 4 B read + 4 B write RMWs)."""
    arcs = 2 * m
    degree = 8 * (n + 1) + 8 * n
    init = 8 * arcs + 4 * st["init_slots_written"] + 4 * n + 32 * f1
    rounds = (32 * (st["frontier_total"] - f1) + 4 * st["bins_read"] + 8 * st["arcs_scanned"]
              + 16 * st["guarded_arcs"])
    # the bucketed edge list of the pull rounds is this implementation's own
    # overhead, not a term of the method: 0 algorithmic bytes
    out = {"degree": degree, "init": init, "rounds": rounds, "edgelist": 0}
    if relabelled:
        out["relabel"] = relabel_bytes(n, m)
    return out


def i2c_bytes(n: int, m: int, st: dict, relabelled: bool = False) -> dict:
    """CntCore / NbrCore ablations, the same 4-byte
    access model: every neighbour-list entry read costs its colidx word and
    the neighbour's estimate (8 B; arcs_scanned counts them), every HINDEX
    evaluation its core read and write (8 B), every active vertex its
    rowptr pair (16 B)."""
    out = {"rounds": 8 * st["arcs_scanned"] + 8 * st["frontier_total"] + 16 * st["alive_scanned"]}
    if relabelled:
        out["relabel"] = relabel_bytes(n, m)
    return out


def relabel_bytes(n: int, m: int) -> int:
    """Internal relabel: degree keys (rowptr 8(n+1), keys+ids 8n), radix sort of
    n (key, id) pairs (4 passes x 16 B), perm/rowptr2 (12n), row copy (rowptr
    16 per row, colidx read + perm gather + colidx2 write = 12 per arc) and the
    final coreness gather (12n)."""
    return 8 * (n + 1) + 8 * n + 64 * n + 12 * n + 16 * n + 12 * 2 * m + 12 * n


def po_bytes(n: int, m: int, st: dict, relabelled: bool = False) -> dict:
    """B_alg = 16n + 4*2m [colidx] + 4*2m [guard reads] + 8*G
    [clamped RMW] + 8*pushes + 4*sum_k |alive_k| + 4n; degree slot = rowptr +
    core + alive list, peel slot = the rest (rowptr of each processed row)."""
    degree = 8 * (n + 1) + 8 * n
    peel = (16 * n + 8 * st["arcs_scanned"] + 8 * st["guarded_arcs"] + 8 * st["pushes"]
            + 4 * st["alive_scanned"])
    out = {"degree": degree, "peel": peel}
    if relabelled:
        out["relabel"] = relabel_bytes(n, m)
    return out


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_slot(config: str, algo: str, slot: str):
    """The committed ncu summary of a kernel slot (profiles/ncu_traffic.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)[config][algo][slot]
    except Exception:
        return {}


def ncu_traffic(config: str, algo: str, slot: str):
    """Per-launch DRAM bytes of a kernel slot from the committed ncu summary."""
    return ncu_slot(config, algo, slot).get("dram_bytes_per_step")


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]
        if not self.lines:  # timed region shorter than the sampling period
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=10).stdout
                self.lines = [ln for ln in out.splitlines() if ln.strip()]
            except Exception:
                pass

    def summary(self):
        if not getattr(self, "lines", None):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except Exception:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
def build_graph(config: str, device):
    import synth
    cfg = synth.CONFIGS[config]
    t0 = time.time()
    rp, ci = cfg.build(device=device)
    if str(device).startswith("cuda"):
        import torch
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
    log(f"[bench] graph {config}: n={rp.numel() - 1} 2m={ci.numel()} built in {time.time() - t0:.1f}s")
    return cfg, rp, ci


def oracle_baseline(rp_np, ci_np, budget_s: float = 12.0, max_runs: int = 5):
    import oracle
    oracle.build_oracle()
    times, core = [], None
    while len(times) < max_runs and (sum(times) < budget_s or not times):
        t0 = time.perf_counter()
        core = oracle.bz(rp_np, ci_np)
        times.append(time.perf_counter() - t0)
    return core, times


def run_reference(args):
    """--impl reference: the CPU oracle (serial BZ) as it stands."""
    import torch
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    dev = torch.device("cuda:0") if torch.cuda.is_available() else torch.device("cpu")
    cfg, rp, ci = build_graph(args.config, dev)
    import synth
    rp_np, ci_np = synth.to_numpy(rp, ci)
    del rp, ci
    import oracle
    oracle.build_oracle()
    n, m = rp_np.size - 1, ci_np.size // 2
    for _ in range(args.warmup):
        oracle.bz(rp_np, ci_np)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.bz(rp_np, ci_np)
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    val = m / t
    sample = f"full {args.config} graph (n={n}, m={m}) per step, serial BZ bucket peel"
    out = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
           "config": {"workload": cfg.note, "config": args.config, "n": n, "m": m, "algo": "oracle_bz"},
           "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
           "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "gpu_launches": 0}
    print(json.dumps(out), flush=True)
    return 0


def time_steps(fn, steps, warmup, stream):
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def bench_single(args):
    import numpy as np
    import torch

    import paper_2402_15253_b200 as pico
    import synth

    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    cfg, rp, ci = build_graph(args.config, dev)
    n, m = rp.numel() - 1, ci.numel() // 2
    deg = (rp[1:] - rp[:-1])
    dmax = int(deg.max().item())
    del deg
    peak, peak_src = hbm_peak()

    results = {}
    algos = [args.algo] + ([a for a in ("histocore", "peelone") if a != args.algo] if args.both else [])
    # Index2core ablations (CntCore, NbrCore; the paper's Table tab:nbrcnthisto) on graphs where they
    # finish in seconds
    if args.ablations == "on" or (args.ablations == "auto" and 2 * m <= (320 << 20)):
        algos += ["cntcore", "nbrcore"]
    algos = list(dict.fromkeys(algos))  # (the main algorithm first, once)
    core_ref = None
    for algo in algos:
        # untimed instrumented run: iteration counts + work counters for B_alg
        st = pico.Stats()
        fs = np.zeros(1 << 16, dtype=np.int64)
        ra = np.zeros(1 << 16, dtype=np.int64)
        core = pico.coreness(rp, ci, algo=algo, flags=pico.F_STATS | args.flags, stats=st,
                             frontier_sizes=fs, round_arcs=ra)
        torch.cuda.synchronize()
        sd = st.to_dict()
        # timed steps (per-kernel CUDA events recorded by the library, PICO_F_TIMING)
        acc = {"ms": {}, "launches": {}, "count": 0}

        def step():
            s2 = pico.Stats()
            pico.coreness(rp, ci, algo=algo, flags=pico.F_TIMING | args.flags, stats=s2, out=core)
            d = s2.to_dict()
            for k, v in d["kernel_ms"].items():
                acc["ms"][k] = acc["ms"].get(k, 0.0) + v
            acc["count"] += d["kernel_count"]

        for _ in range(args.warmup):
            step()
        acc = {"ms": {}, "launches": {}, "count": 0}
        torch.cuda.synchronize()
        with ClockSampler(0) as clk:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                step()
            e1.record(stream)
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        kms = {k: v / args.steps for k, v in acc["ms"].items()}
        rl = "relabel" in kms
        ran = {0: "histocore", 1: "peelone"}.get(sd.get("algo"), algo) if algo == "auto" else algo
        if ran == "histocore":
            byts = hc_bytes(n, m, sd, int(fs[0]) if sd["rounds"] > 0 else 0, rl)
        elif ran == "peelone":
            byts = po_bytes(n, m, sd, rl)
        else:
            byts = i2c_bytes(n, m, sd, rl)
        dom = max(kms, key=kms.get)
        ach = byts.get(dom, 0) / (kms[dom] * 1e-3) / 1e9
        total_b = sum(byts.values())
        results[algo] = {
            "ms": ms, "edges_per_s": m / (ms * 1e-3), "arcs_per_s": 2 * m / (ms * 1e-3),
            "rounds_l2": sd["rounds"], "levels": sd["levels"], "kmax": sd["kmax"],
            "kernel_ms_per_step": kms, "alg_bytes": byts,
            "stats": {k: sd[k] for k in ("frontier_total", "init_slots_written", "arcs_scanned",
                                         "guarded_arcs", "bins_read", "pushes", "alive_scanned",
                                         "segments", "hub_fallbacks", "pull_rounds")},
            "frontier_sizes": [int(x) for x in fs[:min(max(sd["rounds"], sd["levels"]), 64)]],
            "round_arcs": [int(x) for x in ra[:min(sd["rounds"], 64)]] if algo == "histocore" else None,
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s",
                         "frac": ach / peak, "traffic": ncu_traffic(args.config, algo, dom),
                         "peak_source": peak_src,
                         "whole_step_frac": total_b / (ms * 1e-3) / 1e9 / peak,
                         # the second ceiling: L2 throughput of the same kernel, % of
                         # peak, time-weighted over its ncu capture (profiles/ncu_traffic.json)
                         "l2_throughput_pct": ncu_slot(args.config, algo, dom).get("l2_throughput_pct")},
            "gpu_launches": acc["count"] // max(args.steps, 1) * args.steps,
            "clocks": clk.summary(),
        }
        if core_ref is None:
            core_ref = core.cpu().numpy()
        else:
            results[algo]["agrees_with_" + algos[0]] = bool(np.array_equal(core.cpu().numpy(), core_ref))
        log(f"[bench] {algo}: {ms:.3f} ms/step, {m / (ms * 1e-3) / 1e9:.3f} G edges/s, kernels {kms}")

    # end to end through the C ABI with pinned HOST buffers (H2D + D2H inside)
    rp_h = rp.cpu().pin_memory()
    ci_h = ci.cpu().pin_memory()
    out_h = torch.empty(n, dtype=torch.int32).pin_memory()
    rp_np, ci_np, out_np = rp_h.numpy(), ci_h.numpy(), out_h.numpy()
    for _ in range(max(1, args.warmup)):
        pico.coreness_host(rp_np, ci_np, algo=args.algo, out=out_np)
    e2e_steps = max(3, min(args.steps, 10))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        pico.coreness_host(rp_np, ci_np, algo=args.algo, out=out_np)
    e2e_t = (time.perf_counter() - t0) / e2e_steps
    e2e = {"value": m / e2e_t, "unit": UNIT, "ms_per_step": 1e3 * e2e_t,
           "h2d_bytes_per_step": 8 * (n + 1) + 4 * 2 * m, "d2h_bytes_per_step": 4 * n}

    # parity vs the oracle + cpu_baseline (oracle timed on this host, 1 core)
    cpu_baseline, parity = None, "skipped"
    if not args.no_oracle:
        rp_np2, ci_np2 = synth.to_numpy(rp, ci)
        ref, times = oracle_baseline(rp_np2, ci_np2)
        parity = "bit-exact" if np.array_equal(ref, core_ref) and np.array_equal(out_np, ref) else "MISMATCH"
        tb = sum(times) / len(times)
        cpu_baseline = {"value": m / tb, "unit": UNIT, "cores": 1, "kind": "oracle",
                        "sample": f"full {args.config} graph (n={n}, m={m}), serial BZ, {len(times)} runs",
                        "ms": 1e3 * tb}

    main = results[args.algo]
    out = {
        "metric": METRIC, "value": main["edges_per_s"], "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": main["ms"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "int32", "data": "synthetic",
        "config": {"workload": cfg.note, "config": args.config, "algo": args.algo, "n": n, "m": m,
                   "arcs": 2 * m, "d_max": dmax, "kmax": main["kmax"],
                   "l2_flush": "inputs larger than L2 (colidx %.0f MB, histogram %.0f MB > 126 MB)"
                   % (8 * m / 1e6, 8 * m / 1e6)},
        "roofline": main["roofline"],
        "cpu_baseline": cpu_baseline,
        "e2e": e2e,
        "gpu_launches": main["gpu_launches"],
        "clocks": main["clocks"],
        "parity": parity,
        "iterations": {"histocore_l2": results.get("histocore", {}).get("rounds_l2"),
                       "peelone_levels": results.get("peelone", {}).get("levels")},
        "per_algo": results,
    }
    print(json.dumps(out), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--algo", default="histocore", choices=["histocore", "peelone", "auto", "cntcore", "nbrcore"])
    ap.add_argument("--impl", default="pico", choices=["pico", "reference"])
    ap.add_argument("--no-oracle", action="store_true")
    ap.add_argument("--no-both", dest="both", action="store_false")
    ap.add_argument("--ablations", default="auto", choices=["auto", "on", "off"],
                    help="also time CntCore / NbrCore (auto: graphs up to 320 M arcs)")
    ap.add_argument("--flags", type=int, default=0, help="extra PICO_F_* flags (A/B runs)")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "torch"],
                    help="sharded path: NCCL inside libpico (pico_coreness_sharded) or torch.distributed")
    ap.add_argument("--sharded", action="store_true",
                    help="run the sharded path even at one rank (torchrun --nproc-per-node 1)")
    args = ap.parse_args()
    if args.warmup < 3:
        log("[bench] warmup raised to 3 (timing rule)")
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if args.gpus > 1 and world == 0:
        # not launched by torchrun: launch one process per GPU ourselves
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(29500 + os.getpid() % 1000)] + sys.argv
        return subprocess.call(cmd)
    if world > 1 or args.gpus > 1 or args.sharded:
        from bench_sharded import bench_sharded
        return bench_sharded(args)
    return bench_single(args)


if __name__ == "__main__":
    sys.exit(main())
