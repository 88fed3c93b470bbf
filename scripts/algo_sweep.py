"""HistoCore vs PeelOne device time over RMAT scales and initiators (the data
behind PICO_ALGO_AUTO's rule; GPU only).  Prints one line per graph."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_15253_b200 as pico  # noqa: E402
import synth  # noqa: E402


def t_of(rp, ci, algo, reps=5):
    for _ in range(2):
        pico.coreness(rp, ci, algo=algo)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        pico.coreness(rp, ci, algo=algo)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


dev = torch.device("cuda:0")
for abcd, tag in (((0.57, 0.19, 0.19, 0.05), "rmat"), ((0.45, 0.15, 0.15, 0.25), "flat")):
    for scale in (12, 14, 16, 18, 20, 22):
        for ef in (4, 16, 64):
            if scale + ef.bit_length() > 29:
                continue
            rp, ci = synth.rmat(scale, edge_factor=ef, abcd=abcd, seed=scale * 7 + ef, compact=True, device=dev)
            st = pico.Stats()
            pico.coreness(rp, ci, algo="peelone", stats=st)
            hc, po = t_of(rp, ci, "histocore"), t_of(rp, ci, "peelone")
            deg = rp[1:] - rp[:-1]
            print(f"{tag} s{scale} ef{ef} n={rp.numel() - 1} arcs={ci.numel()} dmax={int(deg.max())} "
                  f"kmax={st.kmax} levels={st.levels} hc_ms={hc:.3f} po_ms={po:.3f} ratio={hc / po:.2f}", flush=True)
            del rp, ci, deg
            torch.cuda.empty_cache()
