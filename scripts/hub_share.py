"""Share of the arcs whose neighbour is among the top-K vertices by degree
(the records a per-SM shared-memory hub table would serve in pull rounds)."""
import sys
import torch
sys.path.insert(0, ".")
import bench

for cfg in sys.argv[1:] or ["T"]:
    _, rp, ci = bench.build_graph(cfg, torch.device("cuda"))
    deg = (rp[1:] - rp[:-1])
    M = int(deg.sum())
    ds, _ = torch.sort(deg, descending=True)
    cs = torch.cumsum(ds, 0)
    out = {K: round(float(cs[K - 1]) / M, 3) for K in (8192, 16384, 24576, 32768, 49152, 65536, 131072)}
    print(cfg, "n", rp.numel() - 1, "2m", M, "dmax", int(ds[0]), "top-K arc share", out, flush=True)
    del rp, ci, deg, ds, cs
    torch.cuda.empty_cache()
