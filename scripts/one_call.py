"""One plain (no stats, no timing) library call per algorithm on a config's
graph -- the command ncu profiles.  usage: one_call.py CONFIG [algo ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_15253_b200 as pico  # noqa: E402
import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
algos = sys.argv[2:] or ["histocore", "peelone"]
rp, ci = synth.CONFIGS[cfg].build(device=torch.device("cuda:0"))
torch.cuda.synchronize()
torch.cuda.empty_cache()
for algo in algos:
    pico.coreness(rp, ci, algo=algo)
torch.cuda.synchronize()
print("ok", cfg, algos)
