"""Per-round device-time profile of the persistent HistoCore round kernel
(diagnostic; GPU only).  For each round t: |C_t|, sum of deg over C_t, the
UpdateHisto direction the kernel chose, and the device time of UpdateHisto(t)
and of the SumHisto that builds F_{t+1} (pico_stats_t.round_ns).

    python scripts/round_profile.py --config C2 [--flags 0] [--reps 3]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_15253_b200 as pico  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    rp, ci = synth.CONFIGS[args.config].build(device=dev)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    n, arcs = rp.numel() - 1, ci.numel()
    for _ in range(2):
        pico.coreness(rp, ci, flags=args.flags)
    torch.cuda.synchronize()
    best = None
    for _ in range(args.reps):
        st = pico.Stats()
        fs = np.zeros(1 << 12, dtype=np.int64)
        ra = np.zeros(1 << 12, dtype=np.int64)
        rn = np.zeros(2 << 12, dtype=np.int64)
        pico.coreness(rp, ci, flags=args.flags | pico.F_TIMING, stats=st, frontier_sizes=fs, round_arcs=ra,
                      round_ns=rn)
        torch.cuda.synchronize()
        tot = rn[: 2 * st.rounds].sum()
        if best is None or tot < best[0]:
            best = (tot, st, fs.copy(), ra.copy(), rn.copy())
    _, st, fs, ra, rn = best
    d = st.to_dict()
    print(f"{args.config}: n={n} 2m={arcs} l2={st.rounds} kernel_ms={d['kernel_ms']}")
    print(f"{'t':>3} {'|C_t|':>10} {'arcs(C_t)':>12} {'arcs/2m':>8} {'upd_ms':>8} {'sum_ms':>8}")
    su = ss = 0.0
    for t in range(1, st.rounds + 1):
        u, s = rn[2 * (t - 1)] / 1e6, rn[2 * (t - 1) + 1] / 1e6
        su += u
        ss += s
        print(f"{t:>3} {fs[t - 1]:>10} {ra[t - 1]:>12} {ra[t - 1] / arcs:>8.3f} {u:>8.3f} {s:>8.3f}")
    print(f"total update {su:.3f} ms, sum {ss:.3f} ms")


if __name__ == "__main__":
    main()
