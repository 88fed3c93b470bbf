"""Repeated PeelOne calls (the bench's timed-step call) on one config; reports errors and mismatches."""
import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2402_15253_b200 as pico, synth
cfg, reps = sys.argv[1], int(sys.argv[2])
rp, ci = synth.CONFIGS[cfg].build(device=torch.device("cuda:0"))
ref = pico.coreness(rp, ci, algo="histocore").cpu().numpy()
core = torch.empty(rp.numel() - 1, dtype=torch.int32, device="cuda")
bad = 0
for i in range(reps):
    st = pico.Stats()
    try:
        pico.coreness(rp, ci, algo="peelone", stats=st, out=core)
    except Exception as e:
        print(os.environ.get("PICO_LIB"), cfg, "call", i, "ERROR", e, flush=True)
        sys.exit(3)
    if i % 10 == 0:
        bad += int((core.cpu().numpy() != ref).sum())
print(os.environ.get("PICO_LIB"), cfg, "ok", reps, "calls, mismatches", bad, flush=True)
