#!/usr/bin/env python
"""bench.py -- k-core decomposition throughput on B200 (BASELINE.json metric:
"k-core decomposition edges/sec and ms (1/2/4/8 B200), % of HBM roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config T]
                    [--algo histocore|peelone] [--impl pico|reference]

A step = one coreness computation of the whole graph through the C ABI
(pico_coreness_ex: device-resident CSR in, device-resident coreness out,
workspace allocation included).  value = undirected edges m
/ step time (edges/s).  At T the inputs (colidx 8.4 GB, histogram 8.4 GB)
are far larger than the 126 MB L2; small configs flush L2 between steps.

N = 1: the HistoCore primary kernel on the north-star "1B-edge RMAT" (config
T: RMAT-26, edge factor 16, 2^30 samples), with PeelOne on the
same graph alongside, parity against the serial BZ oracle in the same run,
and the other single-GPU configs (--extras, default C2,C3) timed after it.
roofline.frac = the METHOD's algorithmic bytes of the round kernel (SURVEY
8(d) B_alg with S_t = sum of deg over C_t) / its CUDA-event time / the
measured HBM peak; the implementation's own extra traffic (pull streaming,
edge-list build, compaction) is reported apart as impl_bytes.
N > 1 (torchrun, one process per GPU): sharded HistoCore over a 1-D vertex
partition, value = m / max-over-ranks step time.

--impl reference: the CPU oracle (serial Batagelj-Zaversnik, oracle/) timed on
this box's host cores -- the reference arm of this tier -- on a bounded sample
of the workload (the same RMAT recipe at scale 22) so the run ends in minutes.
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
DEFAULT_CONFIG = "T"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# roofline model: algorithmic bytes per kernel slot (DESIGN.md "Algorithmic
# bytes"; SURVEY 8(d) 4-byte access model, each logical access counted once)
# ---------------------------------------------------------------------------
def hc_bytes(n: int, m: int, st: dict, f1: int, s_method: int, relabelled: bool = False) -> dict:
    """SURVEY 8(d) METHOD bytes: B_alg = 8(n+1) + 4*2m [colidx] + 4*2m [gather
    deg] + 4*W1 [init slots] + 12n [core/oldcore init, initial cnt] + sum_t
    (32|F_t| + 4 bins_t + 8 S_t + 16 G_t), split by kernel slot: degree =
    rowptr + the two estimate arrays; init = colidx + degree gathers + W1 +
    core + the round-1 frontier (32|F_1|); rounds = the per-round terms, with
    S_t = sum_{v in C_t} deg(v) (the method's scanned arcs, ``round_arcs``)
    and G_t = guarded arcs (two 4 B read + 4 B write RMWs).  The arcs a pull
    round streams beyond S_t, the bucketed edge list and the compaction are
    this implementation's own traffic: see ``hc_impl_bytes``."""
    arcs = 2 * m
    degree = 8 * (n + 1) + 8 * n
    init = 8 * arcs + 4 * st["init_slots_written"] + 4 * n + 32 * f1
    rounds = (32 * (st["frontier_total"] - f1) + 4 * st["bins_read"] + 8 * s_method
              + 16 * st["guarded_arcs"])
    return {"degree": degree, "init": init, "rounds": rounds}


def hc_impl_bytes(n: int, m: int, st: dict, s_method: int, relabelled: bool, npass: int) -> dict:
    """Bytes this implementation moves that are NOT terms of the method:
    pull rounds stream every arc of the bucketed edge list (8 B: the u and v
    columns) instead of the rows of C_t; the edge-list build reads colidx
    twice and writes the two columns (plus the row-owner column when
    bucketed); the compaction remaps colidx (relabel_bytes)."""
    arcs = 2 * m
    pull_extra = 8 * max(st["arcs_scanned"] - s_method, 0) + 4 * st["pull_rounds"] * arcs
    out = {"pull_stream_extra": pull_extra}
    if st["pull_rounds"] or npass:
        out["edgelist"] = (24 if npass > 1 else 8) * arcs
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
    """Internal compaction (relabel.cu): bitmap of non-isolated ids (rowptr
    8(n+1)), rowptr2 + inverse map (12 n), the colidx remap (read + write, 8
    B per arc; the rank words are L2-resident) and the coreness map-back (8 n)."""
    return 8 * (n + 1) + 12 * n + 8 * 2 * m + 8 * n


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


# the reference arm's bounded sample of each workload: the same generator
# recipe at a scale whose serial BZ takes a few seconds per step
REF_SAMPLE = {"T": ("rmat", 22, 16 << 22, (0.57, 0.19, 0.19, 0.05), 6, 0.0, False),
              "C4": ("kron", 22, (1_400_000_000 >> 4), (0.57, 0.19, 0.19, 0.05), 4, 0.1, True),
              "C5": ("rmat", 22, 16 << 22, (0.57, 0.19, 0.19, 0.05), 5, 0.0, False)}


def reference_graph(config: str, device):
    """The graph the reference arm times: the config itself when its serial BZ
    takes seconds, else the same recipe at scale 22 (REF_SAMPLE)."""
    import synth
    if config not in REF_SAMPLE:
        cfg, rp, ci = build_graph(config, device)
        return cfg, rp, ci, f"full {config} graph"
    kind, scale, samples, abcd, seed, noise, compact = REF_SAMPLE[config]
    sc = synth.GraphConfig(f"{config}-sample", kind, scale, samples, abcd=abcd, seed=seed, noise=noise,
                           compact=compact)
    rp, ci = sc.build(device=device)
    return synth.CONFIGS[config], rp, ci, (f"{config} recipe at scale {scale} ({samples} samples, seed {seed}): "
                                           "a bounded sample of the workload")


def run_reference(args):
    """--impl reference: the CPU oracle (serial BZ) as it stands, on the host."""
    import torch
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    dev = torch.device("cuda:0") if torch.cuda.is_available() else torch.device("cpu")
    cfg, rp, ci, what = reference_graph(args.config, dev)
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
    sample = f"{what} (n={n}, m={m}) per step, serial BZ bucket peel on 1 host core"
    out = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
           "config": {"workload": cfg.note, "config": args.config, "n": n, "m": m, "algo": "oracle_bz",
                      "sample": what},
           "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
           "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "gpu_launches": 0}
    print(json.dumps(out), flush=True)
    return 0


L2_BYTES = 126 << 20


def timed_steps(fn, steps: int, warmup: int, stream, flush_bytes: int = 0):
    """Run `warmup` untimed steps, then `steps` steps each bracketed by CUDA
    events on `stream`; between timed steps an optional L2 flush (a write of
    `flush_bytes` > L2, outside the event pairs).  Returns the mean step ms."""
    import torch
    for _ in range(warmup):
        fn()
    flush = torch.empty(flush_bytes // 4, dtype=torch.int32, device="cuda") if flush_bytes else None
    torch.cuda.synchronize()
    evs = []
    for _ in range(steps):
        if flush is not None:
            flush.fill_(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in evs) / max(steps, 1)


def measure_algo(pico, rp, ci, algo: str, args, stream, flush_bytes: int, peak: float, with_clocks=True):
    """One algorithm on one device-resident graph: an untimed instrumented run
    (iteration counts, work counters, per-round arcs), a per-kernel pass
    (library CUDA events on the launch stream, PICO_F_TIMING), then the timed
    headline steps WITHOUT instrumentation."""
    import numpy as np
    import torch
    n, m = rp.numel() - 1, ci.numel() // 2
    st = pico.Stats()
    fs = np.zeros(1 << 16, dtype=np.int64)
    ra = np.zeros(1 << 16, dtype=np.int64)
    fcnt = np.zeros(max(n, 1), dtype=np.int32) if algo == "histocore" else None
    core = pico.coreness(rp, ci, algo=algo, flags=pico.F_STATS | args.flags, stats=st,
                         frontier_sizes=fs, round_arcs=ra, frontier_counts=fcnt)
    torch.cuda.synchronize()
    sd = st.to_dict()
    fig3 = fig3_summary(rp, ci, fcnt[:n]) if fcnt is not None else None
    # per-kernel times: a separate instrumented pass (events created per launch slot)
    acc = {"ms": {}, "n": 0}

    def kstep():
        s2 = pico.Stats()
        pico.coreness(rp, ci, algo=algo, flags=pico.F_TIMING | args.flags, stats=s2, out=core)
        for k, v in s2.to_dict()["kernel_ms"].items():
            acc["ms"][k] = acc["ms"].get(k, 0.0) + v
        acc["n"] += 1

    kstep()
    acc = {"ms": {}, "n": 0}
    for _ in range(max(3, min(args.steps, 5))):
        kstep()
    kms = {k: v / acc["n"] for k, v in acc["ms"].items()}
    # headline steps: the plain call, no per-kernel events
    cnt = {"launches": 0}

    def step():
        s3 = pico.Stats()
        pico.coreness(rp, ci, algo=algo, flags=args.flags, stats=s3, out=core)
        cnt["launches"] += s3.kernel_count

    if with_clocks:
        with ClockSampler(torch.cuda.current_device()) as clk:
            ms = timed_steps(step, args.steps, args.warmup, stream, flush_bytes)
        clocks = clk.summary()
    else:
        ms = timed_steps(step, args.steps, args.warmup, stream, flush_bytes)
        clocks = None
    launches = cnt["launches"] // (args.steps + args.warmup) * args.steps
    relabelled = "relabel" in kms
    ran = {0: "histocore", 1: "peelone"}.get(sd.get("algo"), algo) if algo == "auto" else algo
    l2r = sd["rounds"]
    ra_list = [int(x) for x in ra[:l2r]] if ran == "histocore" else None
    impl = {}
    if ran == "histocore":
        s_method = int(sum(ra_list)) if ra_list else 0
        byts = hc_bytes(n, m, sd, int(fs[0]) if l2r > 0 else 0, s_method, relabelled)
        impl = hc_impl_bytes(n, m, sd, s_method, relabelled, 1 if "edgelist" in kms else 0)
    elif ran == "peelone":
        byts = po_bytes(n, m, sd, False)
        if relabelled:
            impl = {"relabel": relabel_bytes(n, m)}
    else:
        byts = i2c_bytes(n, m, sd, False)
        if relabelled:
            impl = {"relabel": relabel_bytes(n, m)}
    dom = max((k for k in kms if k in byts), key=kms.get)
    ach = byts[dom] / (kms[dom] * 1e-3) / 1e9
    total_b = sum(byts.values())
    res = {
        "ms": ms, "edges_per_s": m / (ms * 1e-3), "arcs_per_s": 2 * m / (ms * 1e-3),
        "rounds_l2": sd["rounds"], "levels": sd["levels"], "subrounds": sd["subrounds"], "kmax": sd["kmax"],
        "kernel_ms_per_step": kms, "alg_bytes": byts, "impl_bytes": impl,
        "stats": {k: sd[k] for k in ("frontier_total", "init_slots_written", "arcs_scanned",
                                     "guarded_arcs", "bins_read", "pushes", "alive_scanned",
                                     "segments", "hub_fallbacks", "pull_rounds")},
        "frontier_sizes": [int(x) for x in fs[:min(max(sd["rounds"], sd["levels"]), 4096)]],
        "round_arcs": ra_list,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s",
                     "frac": ach / peak,
                     "whole_step_frac": total_b / (ms * 1e-3) / 1e9 / peak,
                     "whole_step_frac_incl_impl": (total_b + sum(impl.values())) / (ms * 1e-3) / 1e9 / peak},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if fig3 is not None:
        res["fig3"] = fig3
    return core, res


def fig3_summary(rp, ci, fcnt):
    """The paper's Fig 3 measure from the library's per-vertex
    frontier counts (PICO_F_STATS, pico_stats_t.frontier_counts): the share of
    (non-isolated) vertices that are a frontier more than 2 times, and of edges
    read more than 2 / more than 5 times (an edge {u, v} is read once per round
    in which u or v is a frontier: f(u) + f(v) times).  Arcs are counted on
    the GPU in chunks (each undirected edge appears twice, with the same
    count, so arc shares are edge shares)."""
    import torch
    dev = rp.device
    f = torch.from_numpy(fcnt).to(dev)
    deg = rp[1:] - rp[:-1]
    live = deg > 0
    nl = int(live.sum())
    out = {"vertices_frontier_ge1": float(((f >= 1) & live).sum()) / max(nl, 1),
           "vertices_frontier_gt2": float(((f > 2) & live).sum()) / max(nl, 1),
           "vertices_frontier_max": int(f.max()) if f.numel() else 0}
    arcs = ci.numel()
    gt2 = gt5 = 0
    step = 1 << 27
    for s0 in range(0, arcs, step):
        e = torch.arange(s0, min(arcs, s0 + step), dtype=torch.int64, device=dev)
        u = torch.searchsorted(rp, e, right=True) - 1
        acc = f[u] + f[ci[s0:s0 + e.numel()].long()]
        gt2 += int((acc > 2).sum())
        gt5 += int((acc > 5).sum())
        del e, u, acc
    out["edges_read_gt2"] = gt2 / max(arcs, 1)
    out["edges_read_gt5"] = gt5 / max(arcs, 1)
    out["paper_soc_twitter_2010"] = {"vertices_frontier_gt2": 0.189, "edges_read_gt2": 0.88,
                                     "edges_read_gt5": 0.609, "source": "P:228-231"}
    return out


def bench_single(args):
    import numpy as np
    import torch

    import paper_2402_15253_b200 as pico
    import synth

    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    peak, peak_src = hbm_peak()
    cfg, rp, ci = build_graph(args.config, dev)
    n, m = rp.numel() - 1, ci.numel() // 2
    dmax = int((rp[1:] - rp[:-1]).max().item()) if n else 0
    big = 4 * 2 * m > 4 * L2_BYTES
    flush_bytes = 0 if big else 4 * L2_BYTES
    l2_flush = ("none: inputs larger than L2 (colidx %.0f MB + histogram %.0f MB vs 126 MB L2)"
                % (8 * m / 1e6, 8 * m / 1e6)) if big else \
        "L2 flushed between timed steps (504 MB buffer write outside the step events)"

    results = {}
    algos = [args.algo] + ([a for a in ("histocore", "peelone") if a != args.algo] if args.both else [])
    # Index2core ablations (CntCore, NbrCore; the paper's Table tab:nbrcnthisto) on graphs where they
    # finish in seconds
    if args.ablations == "on" or (args.ablations == "auto" and 2 * m <= (320 << 20)):
        algos += ["cntcore", "nbrcore"]
    algos = list(dict.fromkeys(algos))  # (the main algorithm first, once)
    core_ref = None
    for algo in algos:
        core, res = measure_algo(pico, rp, ci, algo, args, stream, flush_bytes, peak)
        res["roofline"]["peak_source"] = peak_src
        res["roofline"]["traffic"] = ncu_traffic(args.config, algo, res["roofline"]["kernel"])
        res["roofline"]["l2_throughput_pct"] = ncu_slot(args.config, algo, res["roofline"]["kernel"]).get(
            "l2_throughput_pct")
        # the binding ceiling of the dense rounds: the SM -> L2 request interface's busy share
        res["roofline"]["l2_request_pct"] = ncu_slot(args.config, algo, res["roofline"]["kernel"]).get(
            "l2_request_pct")
        if core_ref is None:
            core_ref = core.cpu().numpy()
        else:
            res["agrees_with_" + algos[0]] = bool(np.array_equal(core.cpu().numpy(), core_ref))
        results[algo] = res
        log(f"[bench] {args.config} {algo}: {res['ms']:.3f} ms/step, {res['edges_per_s'] / 1e9:.3f} G edges/s, "
            f"frac {res['roofline']['frac']:.3f} (whole step {res['roofline']['whole_step_frac']:.3f}), "
            f"kernels {res['kernel_ms_per_step']}")
        del core
        torch.cuda.empty_cache()

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

    # parity vs the oracle + cpu_baseline (the oracle timed on this host, 1 core)
    cpu_baseline, parity = None, "skipped"
    if not args.no_oracle:
        rp_np2, ci_np2 = synth.to_numpy(rp, ci)
        ref, times = oracle_baseline(rp_np2, ci_np2, budget_s=10.0)
        parity = "bit-exact" if np.array_equal(ref, core_ref) and np.array_equal(out_np, ref) else "MISMATCH"
        tb = sum(times) / len(times)
        cpu_baseline = {"value": m / tb, "unit": UNIT, "cores": 1, "kind": "oracle",
                        "sample": f"full {args.config} graph (n={n}, m={m}), serial BZ, {len(times)} run(s) "
                                  "(also the parity reference)",
                        "ms": 1e3 * tb}
    del rp, ci, rp_h, ci_h
    torch.cuda.empty_cache()

    # the other single-GPU configs: HistoCore and PeelOne timings (parity for these
    # sizes is covered by tests/test_fullsize.py)
    per_config = {}
    for c in [x for x in args.extras.split(",") if x and x != args.config]:
        _, rpc, cic = build_graph(c, dev)
        nc, mc = rpc.numel() - 1, cic.numel() // 2
        fb = 0 if 4 * 2 * mc > 4 * L2_BYTES else 4 * L2_BYTES
        entry = {"n": nc, "m": mc}
        cref = None
        for algo in ("histocore", "peelone"):
            a2 = argparse.Namespace(**vars(args))
            a2.steps, a2.warmup = max(3, min(args.steps, 10)), 3
            core, res = measure_algo(pico, rpc, cic, algo, a2, stream, fb, peak, with_clocks=False)
            cn = core.cpu().numpy()
            if cref is None:
                cref = cn
            entry[algo] = {k: res[k] for k in ("ms", "edges_per_s", "rounds_l2", "levels", "kmax",
                                               "kernel_ms_per_step")}
            entry[algo]["frac"] = res["roofline"]["frac"]
            entry[algo]["whole_step_frac"] = res["roofline"]["whole_step_frac"]
            entry[algo]["kernel"] = res["roofline"]["kernel"]
            if "fig3" in res:
                entry[algo]["fig3"] = {k: v for k, v in res["fig3"].items() if k != "paper_soc_twitter_2010"}
            if algo == "peelone":
                entry[algo]["agrees_with_histocore"] = bool(np.array_equal(cn, cref))
            log(f"[bench] {c} {algo}: {res['ms']:.3f} ms/step, frac {res['roofline']['frac']:.3f}")
            del core
        per_config[c] = entry
        del rpc, cic
        torch.cuda.empty_cache()

    main = results[args.algo]
    out = {
        "metric": METRIC, "value": main["edges_per_s"], "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": main["ms"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "int32", "data": "synthetic",
        "config": {"workload": cfg.note, "config": args.config, "algo": args.algo, "n": n, "m": m,
                   "arcs": 2 * m, "d_max": dmax, "kmax": main["kmax"], "l2_flush": l2_flush},
        "roofline": main["roofline"],
        "cpu_baseline": cpu_baseline,
        "e2e": e2e,
        "gpu_launches": main["gpu_launches"],
        "clocks": main["clocks"],
        "parity": parity,
        "iterations": {"histocore_l2": results.get("histocore", {}).get("rounds_l2"),
                       "peelone_levels": results.get("peelone", {}).get("levels"),
                       "peelone_subrounds": results.get("peelone", {}).get("subrounds")},
        "per_algo": results,
        "per_config": per_config,
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
    ap.add_argument("--extras", default="C2,C3",
                    help="other single-GPU configs timed after the headline (comma list; '' for none)")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "lsa", "torch"],
                    help="sharded path: NCCL inside libpico (pico_coreness_sharded), the same with the "
                         "device-side exchange over NCCL's device API (PICO_F_LSA_EXCHANGE), or torch.distributed")
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
