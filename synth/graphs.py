"""Seeded synthetic graph generators (shared by the oracle tests and the CUDA
path).  This module holds NONE of the method's arithmetic -- it only builds
inputs: symmetric, deduplicated, loop-free CSR graphs (S:27-33,
S:48) with int64 rowptr and int32 colidx.

Every random draw comes from a counter-based 32-bit hash of (seed, stream,
index) evaluated with plain int64 torch ops, so a graph is bit-identical
whether it is generated on the CPU (small test graphs) or on a GPU (bench
sizes) -- ``device`` only chooses where the same integer arithmetic runs.

Recipes:
  * RMAT / Kronecker: each of ``samples`` edges descends ``scale`` levels of a
    2x2 initiator (a, b, c, d) (Graph500 convention: "edge factor" = samples
    per vertex); Kronecker adds a seeded per-level +-noise to the initiator.
    Then a seeded vertex relabel permutation, symmetrize, drop self loops,
    dedup, optional compaction of isolated vertices.
  * Erdos-Renyi G(n, p) and Chung-Lu power law for the property corpus
    (S:463).
  * Named fixtures: the paper's G1 (edges reconstructed in S:51), P_n,
    C_n, K_n, K_{a,b}, stars, K4+pendant, edgeless.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

_M32 = 0xFFFFFFFF


# ----------------------------------------------------------------------------
# counter-based hashing (overflow-free int64 arithmetic on 32-bit values)
# ----------------------------------------------------------------------------
def _mulmod32(x: torch.Tensor, c: int) -> torch.Tensor:
    """(x * c) mod 2^32 for 0 <= x < 2^32 without int64 overflow."""
    lo = c & 0xFFFF
    hi = (c >> 16) & 0xFFFF
    return ((x * lo) + (((x * hi) & 0xFFFF) << 16)) & _M32


def _fmix32(x: torch.Tensor) -> torch.Tensor:
    """MurmurHash3 32-bit finaliser on int64 tensors holding uint32 values."""
    x = x ^ (x >> 16)
    x = _mulmod32(x, 0x85EBCA6B)
    x = x ^ (x >> 13)
    x = _mulmod32(x, 0xC2B2AE35)
    x = x ^ (x >> 16)
    return x


def _fmix32_int(x: int) -> int:
    x &= _M32
    x ^= x >> 16
    x = (x * 0x85EBCA6B) & _M32
    x ^= x >> 13
    x = (x * 0xC2B2AE35) & _M32
    x ^= x >> 16
    return x


def hash_u32(seed: int, stream: int, idx: torch.Tensor) -> torch.Tensor:
    """Uniform uint32 (held in int64) for counter ``idx`` (int64 >= 0)."""
    key = _fmix32_int(_fmix32_int(seed) ^ _fmix32_int(stream * 0x9E3779B9 + 0x7F4A7C15))
    lo = idx & _M32
    hi = idx >> 32
    h = _fmix32(lo ^ key)
    h = _fmix32(h ^ _fmix32((hi + key) & _M32))
    return h


# ----------------------------------------------------------------------------
# CSR construction
# ----------------------------------------------------------------------------
_SORT_LIM = 1 << 30  # torch.sort handles at most INT_MAX elements per call


def csr_from_edges(n: int, src: torch.Tensor, dst: torch.Tensor):
    """Symmetrize, drop self loops, dedup, sort rows ascending -> CSR.
    Returns (rowptr int64[n+1], colidx int32[2m]) on src's device.  Graphs
    with more than 2^30 arcs are sorted in row ranges (same result: the
    global order of the (row, col) keys is the concatenation of the ranges')."""
    dev = src.device
    src = src.to(torch.int64)
    dst = dst.to(torch.int64)
    keep = src != dst
    src, dst = src[keep], dst[keep]
    keys = torch.cat([src * n + dst, dst * n + src])
    del src, dst, keep
    nparts = max(1, -(-keys.numel() // (_SORT_LIM // 2)))
    counts = torch.zeros(n, dtype=torch.int64, device=dev)
    cols = []
    for q in range(nparts):
        lo, hi = n * q // nparts, n * (q + 1) // nparts
        part = keys if nparts == 1 else keys[(keys >= lo * n) & (keys < hi * n)]
        part = torch.unique_consecutive(torch.sort(part).values)
        rows = part // n
        cols.append((part - rows * n).to(torch.int32))
        counts += torch.bincount(rows, minlength=n)
        del part, rows
    del keys
    colidx = cols[0] if len(cols) == 1 else torch.cat(cols)
    del cols
    rowptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    rowptr[1:] = torch.cumsum(counts, 0)
    return rowptr, colidx


def compact_isolated(rowptr: torch.Tensor, colidx: torch.Tensor):
    """Drop degree-0 vertices and renumber the rest in order."""
    deg = rowptr[1:] - rowptr[:-1]
    keep = deg > 0
    newid = (torch.cumsum(keep.to(torch.int64), 0) - 1).to(torch.int32)
    n2 = int(keep.sum().item())
    rp = torch.zeros(n2 + 1, dtype=torch.int64, device=rowptr.device)
    rp[1:] = torch.cumsum(deg[keep], 0)
    ci = torch.empty_like(colidx)
    for s0 in range(0, colidx.numel(), _SORT_LIM):  # gathers in < INT_MAX chunks
        ci[s0:s0 + _SORT_LIM] = newid[colidx[s0:s0 + _SORT_LIM].to(torch.int64)]
    return rp, ci


def _relabel_perm(n: int, seed: int, device) -> torch.Tensor:
    """Seeded permutation of 0..n-1: order vertices by (hash(v), v)."""
    v = torch.arange(n, dtype=torch.int64, device=device)
    keys = (hash_u32(seed, 0x5EED, v) << 32) | v
    order = torch.argsort(keys)
    perm = torch.empty(n, dtype=torch.int64, device=device)
    perm[order] = v
    return perm


def rmat_edges(scale: int, samples: int, abcd=(0.57, 0.19, 0.19, 0.05), seed: int = 1,
               noise: float = 0.0, device="cpu", chunk: int = 1 << 25, first: int = 0):
    """Raw RMAT/Kronecker samples (src, dst) as int64 tensors (before the
    relabel/symmetrize/dedup steps): samples first .. first+samples-1."""
    a, b, c, d = abcd
    tot = a + b + c + d
    a, b, c = a / tot, b / tot, c / tot
    # per-level initiators (Kronecker noise: seeded, deterministic per level)
    thr = []
    for lvl in range(scale):
        if noise > 0.0:
            u = _fmix32_int(seed * 1315423911 + lvl * 2654435761 + 17) / 4294967296.0
            mu = noise * (2.0 * u - 1.0)
            aa = a * (1.0 - 2.0 * mu * b / (a + d)) if a + d > 0 else a
            bb = b * (1.0 + mu)
            cc = c * (1.0 + mu)
            dd = 1.0 - aa - bb - cc
            s = aa + bb + cc + dd
            aa, bb, cc = aa / s, bb / s, cc / s
        else:
            aa, bb, cc = a, b, c
        t1 = int(aa * 4294967296.0)
        t2 = int((aa + bb) * 4294967296.0)
        t3 = int((aa + bb + cc) * 4294967296.0)
        thr.append((t1, t2, t3))
    srcs, dsts = [], []
    for start in range(first, first + samples, chunk):
        cnt = min(chunk, first + samples - start)
        idx = torch.arange(start, start + cnt, dtype=torch.int64, device=device)
        s = torch.zeros(cnt, dtype=torch.int64, device=device)
        t = torch.zeros(cnt, dtype=torch.int64, device=device)
        for lvl in range(scale):
            r = hash_u32(seed, 1000 + lvl, idx)
            t1, t2, t3 = thr[lvl]
            # quadrant: a -> (0,0), b -> (0,1), c -> (1,0), d -> (1,1)
            right = ((r >= t1) & (r < t2)) | (r >= t3)
            down = r >= t2
            s = (s << 1) | down.to(torch.int64)
            t = (t << 1) | right.to(torch.int64)
            del r, right, down
        srcs.append(s)
        dsts.append(t)
        del idx
    return torch.cat(srcs), torch.cat(dsts)


def rmat(scale: int, edge_factor: float = 16, abcd=(0.57, 0.19, 0.19, 0.05), seed: int = 1,
         noise: float = 0.0, compact: bool = False, samples: int | None = None, device="cpu"):
    """RMAT (noise=0) / Kronecker (noise>0) graph as CSR."""
    n = 1 << scale
    if samples is None:
        samples = int(edge_factor * n)
    src, dst = rmat_edges(scale, samples, abcd, seed, noise, device)
    perm = _relabel_perm(n, seed, src.device)
    src = perm[src]
    dst = perm[dst]
    del perm
    rp, ci = csr_from_edges(n, src, dst)
    del src, dst
    if compact:
        rp, ci = compact_isolated(rp, ci)
    return rp, ci


def rmat_rows(scale: int, vb: int, ve: int, edge_factor: float = 16, abcd=(0.57, 0.19, 0.19, 0.05),
              seed: int = 1, noise: float = 0.0, samples: int | None = None, device="cpu",
              chunk: int = 1 << 25):
    """Rows [vb, ve) of ``rmat(...)`` (compact=False) without building the rest:
    (rowptr_local int64[ve-vb+1] with rowptr_local[0] = 0, colidx_local int32
    with global ids) -- the same arrays as slicing the full CSR, generated by
    one rank of a sharded run (C5: RMAT-30, 33 G arcs, 1/P per GPU).  Every
    rank draws all samples (counter-based, so identical on every rank), maps
    them through the seeded relabel, symmetrizes, keeps the arcs whose source
    it owns, then sorts and dedups its own rows."""
    n = 1 << scale
    if samples is None:
        samples = int(edge_factor * n)
    nloc = ve - vb
    perm = _relabel_perm(n, seed, device).to(torch.int32 if n <= (1 << 31) else torch.int64)
    keys = []
    for start in range(0, samples, chunk):
        cnt = min(chunk, samples - start)
        s, t = rmat_edges(scale, cnt, abcd, seed, noise, device, chunk=cnt, first=start)
        s = perm[s].to(torch.int64)
        t = perm[t].to(torch.int64)
        keep = s != t
        s, t = s[keep], t[keep]
        for a, b in ((s, t), (t, s)):  # both arc directions of each edge
            own = (a >= vb) & (a < ve)
            keys.append(((a[own] - vb) << 31) | b[own])
        del s, t, keep
    del perm
    keys = torch.cat(keys) if keys else torch.zeros(0, dtype=torch.int64, device=device)
    counts = torch.zeros(nloc, dtype=torch.int64, device=device)
    cols = []
    nparts = max(1, -(-keys.numel() // (_SORT_LIM // 2)))
    for q in range(nparts):  # sorted in local row ranges (torch.sort takes < 2^31 items)
        lo, hi = nloc * q // nparts, nloc * (q + 1) // nparts
        part = keys if nparts == 1 else keys[(keys >= (lo << 31)) & (keys < (hi << 31))]
        part = torch.unique_consecutive(torch.sort(part).values)
        rows = part >> 31
        cols.append((part & ((1 << 31) - 1)).to(torch.int32))
        counts += torch.bincount(rows, minlength=nloc)
        del part, rows
    del keys
    colidx = cols[0] if len(cols) == 1 else torch.cat(cols)
    rowptr = torch.zeros(nloc + 1, dtype=torch.int64, device=device)
    rowptr[1:] = torch.cumsum(counts, 0)
    return rowptr, colidx


def erdos_renyi(n: int, p: float, seed: int = 1, device="cpu"):
    """G(n, p): each unordered pair {i<j} present iff hash(seed, i*n+j) < p*2^32."""
    if n <= 1:
        return (torch.zeros(n + 1, dtype=torch.int64, device=device),
                torch.zeros(0, dtype=torch.int32, device=device))
    iu = torch.triu_indices(n, n, offset=1, device=device)
    i, j = iu[0].to(torch.int64), iu[1].to(torch.int64)
    thr = int(p * 4294967296.0)
    keep = hash_u32(seed, 77, i * n + j) < thr
    return csr_from_edges(n, i[keep], j[keep])


def chung_lu(n: int, avg_deg: float = 8.0, exponent: float = 2.5, seed: int = 1, device="cpu"):
    """Chung-Lu power-law graph: pair {i<j} present with prob min(1, w_i w_j / W),
    w_i proportional to (i+1)^(-1/(exponent-1))."""
    idx = torch.arange(n, dtype=torch.float64, device=device)
    w = (idx + 1.0) ** (-1.0 / (exponent - 1.0))
    w = w * (avg_deg * n / w.sum())
    W = float(w.sum().item())
    iu = torch.triu_indices(n, n, offset=1, device=device)
    i, j = iu[0].to(torch.int64), iu[1].to(torch.int64)
    prob = torch.clamp(w[i] * w[j] / W, max=1.0)
    thr = (prob * 4294967296.0).to(torch.int64)
    keep = hash_u32(seed, 78, i * n + j) < thr
    return csr_from_edges(n, i[keep], j[keep])


# ----------------------------------------------------------------------------
# fixtures
# ----------------------------------------------------------------------------
G1_EDGES = [(0, 5), (1, 5), (2, 3), (2, 5), (3, 4), (3, 5), (4, 5)]  # S:51 (Fig 1)


def from_edge_list(n: int, edges, device="cpu"):
    if len(edges) == 0:
        return (torch.zeros(n + 1, dtype=torch.int64, device=device),
                torch.zeros(0, dtype=torch.int32, device=device))
    e = torch.tensor(edges, dtype=torch.int64, device=device)
    return csr_from_edges(n, e[:, 0], e[:, 1])


def g1(device="cpu"):
    return from_edge_list(6, G1_EDGES, device)


def path(n, device="cpu"):
    return from_edge_list(n, [(i, i + 1) for i in range(n - 1)], device)


def cycle(n, device="cpu"):
    return from_edge_list(n, [(i, (i + 1) % n) for i in range(n)], device)


def complete(n, device="cpu"):
    return from_edge_list(n, [(i, j) for i in range(n) for j in range(i + 1, n)], device)


def complete_bipartite(a, b, device="cpu"):
    return from_edge_list(a + b, [(i, a + j) for i in range(a) for j in range(b)], device)


def star(leaves, device="cpu"):
    return from_edge_list(leaves + 1, [(0, i) for i in range(1, leaves + 1)], device)


def k4_pendant(device="cpu"):
    return from_edge_list(5, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3), (3, 4)], device)


def edgeless(n, device="cpu"):
    return from_edge_list(n, [], device)


# ----------------------------------------------------------------------------
# named configurations (BASELINE.json configs)
# ----------------------------------------------------------------------------
@dataclass(frozen=True)
class GraphConfig:
    name: str
    kind: str            # "rmat" | "kron"
    scale: int
    samples: int
    abcd: tuple = (0.57, 0.19, 0.19, 0.05)
    seed: int = 1
    noise: float = 0.0
    compact: bool = False
    note: str = ""

    def build(self, device="cpu"):
        return rmat(self.scale, abcd=self.abcd, seed=self.seed, noise=self.noise,
                    compact=self.compact, samples=self.samples, device=device)

    @property
    def n(self) -> int:
        """Vertex count of an uncompacted config (compacted ones: known after the build)."""
        return 1 << self.scale

    def build_rows(self, vb: int, ve: int, device="cpu"):
        """Rows [vb, ve) only (one rank of a sharded run); uncompacted configs
        (compaction renumbers globally)."""
        if self.compact:
            raise ValueError(f"{self.name} is compacted: build it whole and slice")
        return rmat_rows(self.scale, vb, ve, abcd=self.abcd, seed=self.seed, noise=self.noise,
                         samples=self.samples, device=device)


CONFIGS = {
    # configs[0]: RMAT scale-16, edge factor 16, keep isolated, vs CPU oracle
    "C1": GraphConfig("C1", "rmat", 16, 16 << 16, seed=1, note="RMAT-16 ef16 (configs[0])"),
    # configs[1]: LiveJournal-shaped power-law (~4.8M V, ~69M edges)
    "C2": GraphConfig("C2", "rmat", 23, 69_000_000, seed=2, compact=True,
                      note="LiveJournal-shaped RMAT s23, 69M samples, compacted (configs[1])"),
    # configs[2]: Orkut-shaped dense social graph (~3M V, ~117M edges)
    "C3": GraphConfig("C3", "rmat", 22, 117_000_000, abcd=(0.50, 0.20, 0.20, 0.10), seed=3,
                      compact=True, note="Orkut-shaped RMAT s22 (0.5,0.2,0.2,0.1), compacted (configs[2])"),
    # configs[3]: Twitter-shaped Kronecker (~41M V, ~1.4B edges)
    "C4": GraphConfig("C4", "kron", 26, 1_400_000_000, seed=4, noise=0.1, compact=True,
                      note="Twitter-shaped Kronecker s26, 1.4B samples, compacted (configs[3])"),
    # north-star target "1B-edge RMAT": RMAT-26 edge factor 16
    "T": GraphConfig("T", "rmat", 26, 16 << 26, seed=6, note="RMAT-26 ef16 (north-star target)"),
    # configs[4]: RMAT scale-30 -- 8 GPUs only
    "C5": GraphConfig("C5", "rmat", 30, 16 << 30, seed=5, note="RMAT-30 ef16 (configs[4], 8xB200)"),
    # small configs for tests
    "R12": GraphConfig("R12", "rmat", 12, 16 << 12, seed=12, note="RMAT-12 ef16 test graph"),
    "R14": GraphConfig("R14", "rmat", 14, 16 << 14, seed=14, note="RMAT-14 ef16 test graph"),
}


def to_numpy(rowptr: torch.Tensor, colidx: torch.Tensor):
    return rowptr.cpu().numpy().astype(np.int64), colidx.cpu().numpy().astype(np.int32)
