"""Decremental HistoCore timing (GPU only): delete batches of random edges
from a config's graph and time the update against a full recompute of the
reduced graph; the coreness after the last batch is checked against a full
HistoCore run of the reduced graph (itself pinned to the oracle in tests).
Prints one JSON line."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_15253_b200 as pico  # noqa: E402
import synth  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
    dev = torch.device("cuda:0")
    rp, ci = synth.CONFIGS[cfg].build(device=dev)
    n = rp.numel() - 1
    src = torch.repeat_interleave(torch.arange(n, device=dev, dtype=torch.int32), (rp[1:] - rp[:-1]))
    up = src < ci
    eu, ev = src[up], ci[up]
    del src, up
    m = eu.numel()
    g = torch.Generator(device=dev).manual_seed(5)
    perm = torch.randperm(m, device=dev, generator=g)
    out = {"config": cfg, "n": n, "m": m, "batches": []}
    d = pico.DynamicCoreness(rp, ci)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    done = 0
    keep = torch.ones(m, dtype=torch.bool, device=dev)
    for frac in (1e-5, 1e-4, 1e-3, 1e-2):
        k = max(1, int(m * frac))
        idx = perm[done:done + k]
        done += k
        st = pico.Stats()
        fs = np.zeros(1 << 12, dtype=np.int64)
        torch.cuda.synchronize()
        e0.record()
        d.delete_edges(eu[idx], ev[idx], stats=st, frontier_sizes=fs)
        e1.record()
        torch.cuda.synchronize()
        out["batches"].append({"deleted": k, "update_ms": e0.elapsed_time(e1), "rounds": st.rounds,
                               "changed": int(fs[:st.rounds].sum())})
        keep[idx] = False
    # full recompute of the reduced graph
    rrp, rci = synth.graphs.csr_from_edges(n, eu[keep].to(torch.int64), ev[keep].to(torch.int64))
    for _ in range(2):
        ref = pico.coreness(rrp, rci)
    torch.cuda.synchronize()
    e0.record()
    ref = pico.coreness(rrp, rci)
    e1.record()
    torch.cuda.synchronize()
    out["full_recompute_ms"] = e0.elapsed_time(e1)
    out["agrees_with_full_recompute"] = bool(torch.equal(ref, d.coreness()))
    d.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
