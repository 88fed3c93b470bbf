"""paper_2402_15253_b200 -- B200-native k-core decomposition (PICO,
arXiv 2402.15253): HistoCore (Alg 6) and PeelOne (Alg 4, PO-dyn) as
hand-written sm_100a CUDA behind the C ABI of include/pico.h.

Python is a thin ctypes layer (argument marshalling only).  PyTorch supplies
device memory, streams and process groups.  There is no CPU fallback: on a
machine without the built library or without a GPU every compute call raises.

    import paper_2402_15253_b200 as pico
    core = pico.coreness(rowptr_cuda_int64, colidx_cuda_int32, algo="histocore")
"""
from __future__ import annotations

import ctypes

import numpy as np

from ._lib import (ALGOS, F_DEBUG_INVARIANTS, F_L2_PERSIST, F_PREFILTER, F_CLAMP_CAS, F_CLAMP_SUB, F_HOST_LOOP, F_NO_RELABEL, F_PULL_ALWAYS, F_PUSH_ONLY, F_LSA_EXCHANGE,  # noqa: F401
                   F_RELABEL, F_STATS, F_TIMING, F_TINY_TILES, F_VALIDATE, PicoError, Stats, check, header_functions, load)

__all__ = ["coreness", "coreness_host", "clamp_hammer", "workspace_bytes", "DynamicCoreness", "PicoError", "Stats", "load",
           "F_VALIDATE", "F_STATS", "F_TIMING", "F_HOST_LOOP", "F_CLAMP_SUB", "F_TINY_TILES",
           "F_PUSH_ONLY", "F_PULL_ALWAYS", "F_RELABEL", "F_NO_RELABEL", "F_CLAMP_CAS", "F_PREFILTER", "F_L2_PERSIST", "F_LSA_EXCHANGE"]


def _algo(algo) -> int:
    if isinstance(algo, str):
        if algo not in ALGOS:
            raise ValueError(f"unknown algo {algo!r}; expected one of {sorted(ALGOS)}")
        return ALGOS[algo]
    return int(algo)


def _host_i64(name, a):
    """A caller-supplied host counter array: int64, C-contiguous, writable
    (the library writes up to a.size entries through it)."""
    if not isinstance(a, np.ndarray) or a.dtype != np.int64 or not a.flags["C_CONTIGUOUS"] or not a.flags["WRITEABLE"]:
        raise TypeError(f"{name} must be a writable C-contiguous int64 numpy array")
    return a


def workspace_bytes(n: int, m: int, algo="histocore", flags: int = 0) -> int:
    return int(load().pico_workspace_bytes(n, m, _algo(algo), flags))


def coreness(rowptr, colidx, algo="histocore", flags: int = 0, out=None, workspace=None,
             stats: Stats | None = None, frontier_sizes=None, round_arcs=None, round_ns=None, stream=None,
             frontier_counts=None):
    """Coreness of every vertex of a symmetric deduplicated CSR graph held in
    device memory (``pico_coreness_ex``).

    rowptr: int64 CUDA tensor [n+1]; colidx: int32 CUDA tensor [2m].
    Returns an int32 CUDA tensor [n].  ``stats`` (a :class:`Stats`) is filled
    in place; ``frontier_sizes`` an optional int64 numpy array receiving
    |F_t| per round (HistoCore) or vertices per level (PeelOne);
    ``round_arcs`` / ``round_ns`` (2 entries per round: UpdateHisto, SumHisto
    device ns) optional int64 numpy arrays for HistoCore.  ``frontier_counts``
    (HistoCore, needs PICO_F_STATS): an optional int32 numpy array of >= n
    entries receiving each vertex's number of frontier rounds (the paper's
    Fig 3 measure).
    """
    import torch
    lib = load()
    if not (rowptr.is_cuda and colidx.is_cuda):
        raise ValueError("rowptr and colidx must be CUDA tensors (no CPU fallback)")
    if rowptr.dtype != torch.int64 or colidx.dtype != torch.int32:
        raise TypeError("rowptr must be int64 and colidx int32")
    rowptr = rowptr.contiguous()
    colidx = colidx.contiguous()
    n = rowptr.numel() - 1
    arcs = colidx.numel()
    if arcs % 2:
        raise ValueError("colidx length must be even (2m arcs of a symmetric graph)")
    m = arcs // 2
    if colidx.device != rowptr.device:
        raise ValueError("rowptr and colidx must be on the same device")
    if out is None:
        out = torch.empty(max(n, 0), dtype=torch.int32, device=rowptr.device)
    elif (not isinstance(out, torch.Tensor) or out.dtype != torch.int32 or out.device != rowptr.device
          or not out.is_contiguous() or out.numel() < n):
        raise ValueError(f"out must be a contiguous int32 tensor of >= {n} elements on {rowptr.device}")
    if stream is None:
        stream = torch.cuda.current_stream(rowptr.device)
    ws_ptr, ws_bytes = None, 0
    if workspace is not None:
        ws_ptr, ws_bytes = workspace.data_ptr(), workspace.numel() * workspace.element_size()
    st = stats
    if frontier_counts is not None:
        if not (isinstance(frontier_counts, np.ndarray) and frontier_counts.dtype == np.int32
                and frontier_counts.flags.c_contiguous and frontier_counts.size >= n):
            raise ValueError(f"frontier_counts must be a C-contiguous int32 numpy array of >= {n} entries")
        if st is None:
            st = Stats()
        st.frontier_counts = frontier_counts.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        st.frontier_counts_cap = frontier_counts.size
    if frontier_sizes is None and (round_arcs is not None or round_ns is not None):
        raise ValueError("round_arcs / round_ns need frontier_sizes (their capacity is its size)")
    if frontier_sizes is not None:
        if st is None:
            st = Stats()
        _host_i64("frontier_sizes", frontier_sizes)
        st.frontier_sizes = frontier_sizes.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
        st.frontier_sizes_cap = frontier_sizes.size
        if round_arcs is not None:
            _host_i64("round_arcs", round_arcs)
            if round_arcs.size < frontier_sizes.size:
                raise ValueError("round_arcs must hold at least frontier_sizes.size entries")
            st.round_arcs = round_arcs.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
        if round_ns is not None:
            _host_i64("round_ns", round_ns)
            if round_ns.size < 2 * frontier_sizes.size:
                raise ValueError("round_ns must hold at least 2 * frontier_sizes.size entries")
            st.round_ns = round_ns.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
    with torch.cuda.device(rowptr.device):
        rc = lib.pico_coreness_ex(rowptr.data_ptr(), colidx.data_ptr() if arcs else None, n, m, _algo(algo),
                                  out.data_ptr() if n > 0 else None, ctypes.c_void_p(stream.cuda_stream), flags,
                                  ws_ptr, ws_bytes, ctypes.byref(st) if st is not None else None)
    check(rc)
    return out


def coreness_host(rowptr: np.ndarray, colidx: np.ndarray, algo="histocore", flags: int = 0, out=None,
                  stats: Stats | None = None, stream=None) -> np.ndarray:
    """End-to-end call on HOST arrays (``pico_coreness_host``): H2D copies,
    the CUDA path, D2H of the coreness -- all inside the library call."""
    lib = load()
    rp = np.ascontiguousarray(rowptr, dtype=np.int64)
    ci = np.ascontiguousarray(colidx, dtype=np.int32)
    n = rp.size - 1
    m = ci.size // 2
    if out is None:
        out = np.empty(max(n, 0), dtype=np.int32)
    elif (not isinstance(out, np.ndarray) or out.dtype != np.int32 or not out.flags["C_CONTIGUOUS"]
          or not out.flags["WRITEABLE"] or out.size < n):
        raise ValueError(f"out must be a writable C-contiguous int32 numpy array of >= {n} elements")
    sptr = ctypes.c_void_p(stream.cuda_stream) if stream is not None else None
    rc = lib.pico_coreness_host(rp.ctypes.data, ci.ctypes.data if ci.size else None, n, m, _algo(algo),
                                out.ctypes.data if n > 0 else None, sptr, flags,
                                ctypes.byref(stats) if stats is not None else None)
    check(rc)
    return out


def clamp_hammer(mode: int, d: int, k: int, c: int, stream=None):
    """``pico_clamp_hammer``: c concurrent device threads apply PeelOne's
    clamped decrement atomicSub>=k to one cell holding d at level k,
    in clamp implementation ``mode`` (0 default, 1 sub + repair, 2 CAS).
    Returns (final value, calls that saw old > k, calls that saw k + 1)."""
    lib = load()
    fin = ctypes.c_int32()
    gt = ctypes.c_int64()
    k1 = ctypes.c_int64()
    sptr = ctypes.c_void_p(stream.cuda_stream) if stream is not None else None
    check(lib.pico_clamp_hammer(mode, d, k, c, ctypes.byref(fin), ctypes.byref(gt), ctypes.byref(k1), sptr))
    return fin.value, gt.value, k1.value


class DynamicCoreness:
    """Decremental HistoCore (include/pico_dyn.h): the coreness of a graph
    kept up to date under batches of edge deletions, reusing the persistent
    per-vertex histograms instead of recomputing from scratch.

        d = pico.DynamicCoreness(rowptr, colidx)      # device CSR
        d.delete_edges(src, dst)                      # int32 CUDA tensors
        core = d.coreness()
    """

    def __init__(self, rowptr, colidx, flags: int = 0, stats: Stats | None = None, stream=None):
        import torch
        self.lib = load()
        if not (rowptr.is_cuda and colidx.is_cuda):
            raise ValueError("rowptr and colidx must be CUDA tensors (no CPU fallback)")
        self.dev = rowptr.device
        self.n = rowptr.numel() - 1
        self.stream = stream or torch.cuda.current_stream(self.dev)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.dev):
            check(self.lib.pico_dyn_create(rowptr.contiguous().data_ptr(),
                                           colidx.contiguous().data_ptr() if colidx.numel() else None,
                                           self.n, colidx.numel() // 2, flags,
                                           ctypes.c_void_p(self.stream.cuda_stream),
                                           ctypes.byref(stats) if stats is not None else None, ctypes.byref(h)))
        self.h = h

    def coreness(self, out=None):
        import torch
        if out is None:
            out = torch.empty(self.n, dtype=torch.int32, device=self.dev)
        check(self.lib.pico_dyn_coreness(self.h, out.data_ptr()))
        return out

    def delete_edges(self, src, dst, stats: Stats | None = None, frontier_sizes=None):
        """Delete undirected edges {src[i], dst[i]} (pico_dyn_delete_edges)."""
        return self._update(self.lib.pico_dyn_delete_edges, src, dst, stats, frontier_sizes)

    def insert_edges(self, src, dst, stats: Stats | None = None, frontier_sizes=None):
        """Insert undirected edges {src[i], dst[i]} (pico_dyn_insert_edges)."""
        return self._update(self.lib.pico_dyn_insert_edges, src, dst, stats, frontier_sizes)

    def _update(self, fn, src, dst, stats, frontier_sizes):
        import torch
        if src.numel() != dst.numel():
            raise ValueError(f"src and dst must have the same length ({src.numel()} != {dst.numel()})")
        # the copies run on the handle's stream, which the library uses
        with torch.cuda.stream(self.stream):
            src = src.to(device=self.dev, dtype=torch.int32).contiguous()
            dst = dst.to(device=self.dev, dtype=torch.int32).contiguous()
        st = stats
        if frontier_sizes is not None:
            st = st or Stats()
            _host_i64("frontier_sizes", frontier_sizes)
            st.frontier_sizes = frontier_sizes.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
            st.frontier_sizes_cap = frontier_sizes.size
        check(fn(self.h, src.data_ptr() if src.numel() else None, dst.data_ptr() if dst.numel() else None,
                 src.numel(), ctypes.byref(st) if st is not None else None))
        return st

    def close(self):
        if getattr(self, "h", None):
            check(self.lib.pico_dyn_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
