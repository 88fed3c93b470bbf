"""Experiment (not part of the product): how much would a degree-ordered
vertex layout help HistoCore / PeelOne on a large RMAT graph?  The graph is
relabelled in torch outside the timed region:
  rank r = position of v in degree-descending order (isolated vertices last);
  id(r)  = superblock-local stride permutation (SB ranks per superblock,
           consecutive ranks placed STRIDE ids apart) so that the hottest
           vertices are compact at the MB scale but never share an L2 line /
           slice.
Prints per-kernel times for the original and relabelled graphs."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2402_15253_b200 as pico  # noqa: E402
import synth  # noqa: E402


def spread_perm(n2, sb=1 << 20, stride=2048):
    r = torch.arange(n2, dtype=torch.int64, device="cuda")
    blk = r // sb
    rr = r % sb
    size = torch.clamp(n2 - blk * sb, max=sb)
    g = (size + stride - 1) // stride
    return blk * sb + (rr % g) * stride + rr // g  # may leave gaps inside the last block


def relabel(rp, ci, mode):
    n = rp.numel() - 1
    deg = rp[1:] - rp[:-1]
    order = torch.argsort(-deg * (n + 1) + torch.arange(n, device="cuda"))  # deg desc, id asc
    n2 = int((deg > 0).sum().item())
    rank = torch.empty(n, dtype=torch.int64, device="cuda")
    rank[order] = torch.arange(n, dtype=torch.int64, device="cuda")
    if mode == "spread":
        pos = spread_perm(n2)
        newid = torch.full((n,), -1, dtype=torch.int64, device="cuda")
        live = rank < n2
        newid[live] = pos[rank[live]]
        nn = int(pos.max().item()) + 1
    else:
        newid = torch.where(rank < n2, rank, torch.full_like(rank, -1))
        nn = n2
    src = torch.repeat_interleave(torch.arange(n, device="cuda"), deg)
    s2 = newid[src]
    del src
    d2 = newid[ci.to(torch.int64)]
    keys = s2 * nn + d2
    del s2, d2
    keys = torch.sort(keys).values
    rows = keys // nn
    ci2 = (keys - rows * nn).to(torch.int32)
    del keys
    cnt = torch.bincount(rows, minlength=nn)
    del rows
    rp2 = torch.zeros(nn + 1, dtype=torch.int64, device="cuda")
    rp2[1:] = torch.cumsum(cnt, 0)
    torch.cuda.empty_cache()
    return rp2, ci2


def run(rp, ci, algo, flags=0, reps=3):
    st = pico.Stats()
    out = None
    for _ in range(2):
        out = pico.coreness(rp, ci, algo=algo, flags=flags | pico.F_TIMING, stats=st)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        out = pico.coreness(rp, ci, algo=algo, flags=flags | pico.F_TIMING, stats=st)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t) / reps * 1e3
    return ms, {k: round(v, 1) for k, v in st.to_dict()["kernel_ms"].items()}, out


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "T"
    rp, ci = synth.CONFIGS[cfg].build(device=torch.device("cuda"))
    torch.cuda.empty_cache()
    for algo in ("histocore", "peelone"):
        ms, k, ref = run(rp, ci, algo)
        print(cfg, "original", algo, "%.1f ms" % ms, k, flush=True)
        ref_hist = torch.bincount(ref.to(torch.int64))
        for mode in ("degree", "spread"):
            rp2, ci2 = relabel(rp, ci, mode)
            ms, k, out = run(rp2, ci2, algo)
            same = torch.equal(torch.bincount(out.to(torch.int64))[1:], ref_hist[1:])
            print(cfg, mode, algo, "%.1f ms" % ms, k, "coreness histogram equal:", same, flush=True)
            del rp2, ci2
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
