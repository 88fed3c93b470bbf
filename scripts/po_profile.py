"""PeelOne iteration profile (diagnostic; GPU only): levels, BSP sub-rounds,
alive-list work and device time on a config's graph."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_15253_b200 as pico  # noqa: E402
import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rp, ci = synth.CONFIGS[cfg].build(device=torch.device("cuda:0"))
torch.cuda.synchronize()
torch.cuda.empty_cache()
for _ in range(2):
    pico.coreness(rp, ci, algo="peelone", flags=flags)
st = pico.Stats()
fs = np.zeros(1 << 16, dtype=np.int64)
pico.coreness(rp, ci, algo="peelone", flags=flags | pico.F_STATS, stats=st, frontier_sizes=fs)
d = st.to_dict()
st2 = pico.Stats()
pico.coreness(rp, ci, algo="peelone", flags=flags | pico.F_TIMING, stats=st2)
torch.cuda.synchronize()
print(cfg, "levels", st.levels, "subrounds", st.subrounds, "kmax", st.kmax, "alive_scanned", d["alive_scanned"],
      "arcs", d["arcs_scanned"], "guarded", d["guarded_arcs"], "pushes", d["pushes"], "segments", d["segments"],
      "ms", st2.to_dict()["kernel_ms"])
sizes = fs[:st.levels]
print("level sizes: first", sizes[:10].tolist(), "median", int(np.median(sizes)), "levels < 100 vertices:",
      int((sizes < 100).sum()))
