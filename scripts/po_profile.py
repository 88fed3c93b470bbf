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
fs2 = np.zeros(1 << 16, dtype=np.int64)
rn = np.zeros(2 << 16, dtype=np.int64)
pico.coreness(rp, ci, algo="peelone", flags=flags | pico.F_TIMING, stats=st2, frontier_sizes=fs2, round_ns=rn)
torch.cuda.synchronize()
print(cfg, "levels", st.levels, "subrounds", st.subrounds, "kmax", st.kmax, "alive_scanned", d["alive_scanned"],
      "arcs", d["arcs_scanned"], "guarded", d["guarded_arcs"], "pushes", d["pushes"], "segments", d["segments"],
      "ms", st2.to_dict()["kernel_ms"])
sizes = fs[:st.levels]
print("level sizes: first", sizes[:10].tolist(), "median", int(np.median(sizes)), "levels < 100 vertices:",
      int((sizes < 100).sum()))
nl = int((rn[0::2] > 0).sum())
M40 = (1 << 40) - 1
scan, drain = (rn[0:2 * nl:2] & M40) / 1e3, (rn[1:2 * nl:2] & M40) / 1e3
kk = rn[0:2 * nl:2] >> 40
core = pico.coreness(rp, ci, algo="peelone").cpu().numpy()
deg = (rp[1:] - rp[:-1]).cpu().numpy()
arcs_at = np.bincount(core, weights=deg, minlength=int(core.max()) + 2)
cnt_at = np.bincount(core, minlength=int(core.max()) + 2)
subs = rn[1:2 * nl:2] >> 40
print(f"scanned levels {nl}: scan total {scan.sum() / 1e3:.3f} ms, drain total {drain.sum() / 1e3:.3f} ms; "
      f"per level scan median {np.median(scan):.1f} us, drain median {np.median(drain):.1f} us")
order = np.argsort(-(scan + drain))[:12]
print("slowest levels (index, k, vertices, arcs, scan us, drain us, sub-rounds):",
      [(int(i), int(kk[i]), int(cnt_at[kk[i]]), int(arcs_at[kk[i]]), round(float(scan[i]), 1), round(float(drain[i]), 1),
        int(subs[i])) for i in order])
q = [0, 10, 20, 50, 100, 200, nl]
print("cumulative by level index:", [(q[i], q[i + 1], round(float((scan[q[i]:q[i + 1]] + drain[q[i]:q[i + 1]]).sum() / 1e3), 3))
                                     for i in range(len(q) - 1) if q[i] < nl])
