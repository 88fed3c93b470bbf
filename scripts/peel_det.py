import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2402_15253_b200 as pico, synth, oracle
rp, ci = synth.CONFIGS["T"].build(device=torch.device("cuda:0"))
ref = None
for lib in sys.argv[1:]:
    pass
core_h = pico.coreness(rp, ci, algo="histocore").cpu().numpy()
for i in range(3):
    cp = pico.coreness(rp, ci, algo="peelone").cpu().numpy()
    bad = np.flatnonzero(cp != core_h)
    print(os.environ.get("PICO_LIB", "default"), "run", i, "mismatches", bad.size, bad[:3], flush=True)
