"""Search for the smallest graph on which a PeelOne build disagrees with HistoCore (diagnostic)."""
import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2402_15253_b200 as pico, synth
dev = torch.device("cuda:0")
for scale in range(12, 25):
    for ef in (8, 16, 32):
        for seed in (1, 2, 3):
            rp, ci = synth.rmat(scale, ef, seed=seed, compact=True, device=dev)
            h = pico.coreness(rp, ci, algo="histocore").cpu().numpy()
            p = pico.coreness(rp, ci, algo="peelone").cpu().numpy()
            bad = np.flatnonzero(h != p)
            if bad.size:
                print("FAIL scale", scale, "ef", ef, "seed", seed, "n", rp.numel() - 1, "bad", bad.size, bad[:4], h[bad[:4]], p[bad[:4]], flush=True)
    print("scale", scale, "done", flush=True)
