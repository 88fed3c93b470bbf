"""TEST INFRASTRUCTURE ONLY -- ctypes bindings to oracle/oracle.c plus tiny
pure-Python references.  See oracle/__init__.py for who may import this.

Every function cites the passage of PAPER.md ("P:<line>") or SPEC.md
("S:<line>") it follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_I64P = ctypes.POINTER(ctypes.c_int64)
_I32P = ctypes.POINTER(ctypes.c_int32)


def build_oracle(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain -O2, single thread)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build_oracle())
        lib.oracle_bz.argtypes = [_I64P, _I32P, ctypes.c_int64, _I32P]
        lib.oracle_bz.restype = ctypes.c_int
        lib.oracle_hindex.argtypes = [_I32P, ctypes.c_int64]
        lib.oracle_hindex.restype = ctypes.c_int64
        lib.oracle_jacobi_rounds.argtypes = [_I64P, _I32P, ctypes.c_int64, _I32P, _I64P, ctypes.c_int64]
        lib.oracle_jacobi_rounds.restype = ctypes.c_int64
        lib.oracle_frontier_counts.argtypes = [_I64P, _I32P, ctypes.c_int64, _I32P,
                                               ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
        lib.oracle_frontier_counts.restype = ctypes.c_int64
        lib.oracle_peel_levels.argtypes = [_I64P, _I32P, ctypes.c_int64, _I32P, _I64P, _I64P]
        lib.oracle_peel_levels.restype = ctypes.c_int64
        lib.oracle_kcore_check.argtypes = [_I64P, _I32P, ctypes.c_int64, _I32P]
        lib.oracle_brute.argtypes = [ctypes.c_int64, ctypes.c_void_p, _I32P]
        lib.oracle_brute.restype = ctypes.c_int
        lib.oracle_exhaustive.argtypes = [ctypes.c_int64]
        lib.oracle_exhaustive.restype = ctypes.c_int64
        lib.oracle_kcore_check.restype = ctypes.c_int
        _lib = lib
    return _lib


def _csr(rowptr, colidx):
    rp = np.ascontiguousarray(np.asarray(rowptr, dtype=np.int64))
    ci = np.ascontiguousarray(np.asarray(colidx, dtype=np.int32))
    if ci.size == 0:
        ci = np.zeros(1, dtype=np.int32)  # valid pointer for empty graphs
    return rp, ci


def bz(rowptr, colidx) -> np.ndarray:
    """Coreness by the BZ bin-sort peel."""
    rp, ci = _csr(rowptr, colidx)
    n = rp.size - 1
    core = np.zeros(max(n, 1), dtype=np.int32)
    if n > 0 and _load().oracle_bz(rp.ctypes.data_as(_I64P), ci.ctypes.data_as(_I32P), n,
                                   core.ctypes.data_as(_I32P)) != 0:
        raise MemoryError("oracle_bz allocation failed")
    return core[:n]


def hindex(values: Sequence[int]) -> int:
    """HINDEX by its definition (Alg 2)."""
    a = np.ascontiguousarray(np.asarray(values, dtype=np.int32))
    if a.size == 0:
        return 0
    return int(_load().oracle_hindex(a.ctypes.data_as(_I32P), a.size))


def hindex_sorted(values: Sequence[int]) -> int:
    """Textbook h-index (Hirsch): sort descending, h = #{i : x_(i) >= i}
    (1-based).  An independent formulation used only to pin ``hindex``."""
    xs = sorted((int(x) for x in values), reverse=True)
    h = 0
    for i, x in enumerate(xs, start=1):
        if x >= i:
            h = i
    return h


def jacobi_rounds(rowptr, colidx, max_record: int = 1 << 16):
    """Synchronous Index2core sweeps from core = deg (Alg 2).
    Returns (fixed point, l2, [|F_1|, |F_2|, ...])."""
    rp, ci = _csr(rowptr, colidx)
    n = rp.size - 1
    core = np.zeros(max(n, 1), dtype=np.int32)
    fs = np.zeros(max_record, dtype=np.int64)
    if n == 0:
        return core[:0], 0, []
    l2 = _load().oracle_jacobi_rounds(rp.ctypes.data_as(_I64P), ci.ctypes.data_as(_I32P), n,
                                      core.ctypes.data_as(_I32P), fs.ctypes.data_as(_I64P), max_record)
    if l2 < 0:
        raise MemoryError("oracle_jacobi_rounds allocation failed")
    return core[:n], int(l2), [int(x) for x in fs[: min(l2, max_record)]]


def frontier_counts(rowptr, colidx):
    """The paper's Fig 3 measure on the synchronous sweeps:
    returns (fcount, l2, nbr_unchanged, nbr_total) -- fcount[v] = the sweeps
    in which v is a frontier (an edge {u, v} is read fcount[u] + fcount[v]
    times), and the frontier-neighbour pairs whose neighbour's estimate stays
    unchanged in the next sweep, out of all such pairs."""
    rp, ci = _csr(rowptr, colidx)
    n = rp.size - 1
    fc = np.zeros(max(n, 1), dtype=np.int32)
    un = ctypes.c_int64(0)
    tot = ctypes.c_int64(0)
    if n == 0:
        return fc[:0], 0, 0, 0
    l2 = _load().oracle_frontier_counts(rp.ctypes.data_as(_I64P), ci.ctypes.data_as(_I32P), n,
                                        fc.ctypes.data_as(_I32P), ctypes.byref(un), ctypes.byref(tot))
    if l2 < 0:
        raise MemoryError("oracle_frontier_counts allocation failed")
    return fc[:n], int(l2), int(un.value), int(tot.value)


def peel_levels(rowptr, colidx):
    """Level-synchronous PeelOne-style peel (Alg 4, clamp P:273).
    Returns (coreness, kmax, non-empty levels, BSP sub-rounds)."""
    rp, ci = _csr(rowptr, colidx)
    n = rp.size - 1
    core = np.zeros(max(n, 1), dtype=np.int32)
    lv = ctypes.c_int64(0)
    sr = ctypes.c_int64(0)
    if n == 0:
        return core[:0], 0, 0, 0
    kmax = _load().oracle_peel_levels(rp.ctypes.data_as(_I64P), ci.ctypes.data_as(_I32P), n,
                                      core.ctypes.data_as(_I32P), ctypes.byref(lv), ctypes.byref(sr))
    if kmax < 0:
        raise MemoryError("oracle_peel_levels allocation failed")
    return core[:n], int(kmax), int(lv.value), int(sr.value)


def kcore_check(rowptr, colidx, core) -> bool:
    """Definition check: every v has >= core[v] neighbours with core >= core[v]."""
    rp, ci = _csr(rowptr, colidx)
    c = np.ascontiguousarray(np.asarray(core, dtype=np.int32))
    n = rp.size - 1
    if n == 0:
        return True
    return bool(_load().oracle_kcore_check(rp.ctypes.data_as(_I64P), ci.ctypes.data_as(_I32P), n,
                                           c.ctypes.data_as(_I32P)))


def brute_coreness(n: int, edges) -> list:
    """Repeated removal of a minimum-degree vertex (Peel, Alg 1 P:118-130;
    S:173): coreness(v) = the running maximum of the minimum degree at the
    time v is removed.  O(n^2); tiny graphs only."""
    adj = [set() for _ in range(n)]
    for u, v in edges:
        if u != v:
            adj[u].add(v)
            adj[v].add(u)
    alive = set(range(n))
    deg = {v: len(adj[v]) for v in range(n)}
    core = [0] * n
    k = 0
    while alive:
        v = min(alive, key=lambda x: (deg[x], x))
        k = max(k, deg[v])
        core[v] = k
        alive.remove(v)
        for u in adj[v]:
            if u in alive:
                deg[u] -= 1
    return core


def histogram_state(rowptr, colidx, core, v: int) -> dict:
    """The HistoCore histogram invariant for vertex v rebuilt from a core
    array by brute force (Alg 6): bins j < core[v] hold
    |{u in nbr(v): core[u] == j}|, the cap bin core[v] holds
    |{u in nbr(v): core[u] >= core[v]}| (= cnt); higher bins are stale."""
    rp = np.asarray(rowptr)
    ci = np.asarray(colidx)
    c = np.asarray(core)
    cv = int(c[v])
    nb = c[ci[rp[v]:rp[v + 1]]]
    out = {j: int(np.sum(nb == j)) for j in range(1, cv)}
    out[cv] = int(np.sum(nb >= cv))
    return out


def brute_c(n: int, edges) -> list:
    """oracle_brute (C): repeated minimum-degree removal on an adjacency matrix."""
    lib = _load()
    adj = np.zeros((n, n), dtype=np.uint8)
    for u, v in edges:
        if u != v:
            adj[u, v] = adj[v, u] = 1
    out = np.zeros(max(n, 1), dtype=np.int32)
    if lib.oracle_brute(n, adj.ctypes.data, out.ctypes.data_as(_I32P)) != 0:
        raise ValueError("oracle_brute: n must be <= 64")
    return out[:n].tolist()


def exhaustive_mismatches(n: int) -> int:
    """Graphs on n vertices (all 2^(n(n-1)/2) of them) where BZ and the C brute
    force differ."""
    return int(_load().oracle_exhaustive(n))
