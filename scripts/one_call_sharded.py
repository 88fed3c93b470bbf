"""One sharded HistoCore call (NCCL inside libpico, one rank) on a config's
graph -- for ncu launch lists of the sharded kernels."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_15253_b200 import sharded  # noqa: E402
import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
rp, ci = synth.CONFIGS[cfg].build(device=torch.device("cuda:0"))
torch.cuda.synchronize()
comm = sharded.NcclComm(nranks=1, rank=0)
n, m = rp.numel() - 1, ci.numel() // 2
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    run = sharded.coreness_sharded_nccl(rp, ci, n, m, 0, comm)
torch.cuda.synchronize()
comm.close()
print("ok", cfg, run.rounds)
