"""ctypes binding of libpico.so -- argument marshalling only.  Every step of
the coreness computation runs in the library's CUDA kernels; there is no
Python or CPU fallback: if the library cannot be loaded, or no GPU is
present, calls raise."""
from __future__ import annotations

import ctypes
import os
import re

from .build import INCLUDE, LIB

ALGOS = {"histocore": 0, "peelone": 1, "auto": 2, "cntcore": 3, "nbrcore": 4}

F_VALIDATE = 1
F_STATS = 2
F_TIMING = 4
F_HOST_LOOP = 8
F_CLAMP_SUB = 16
F_TINY_TILES = 32
F_PUSH_ONLY = 64
F_PULL_ALWAYS = 128
F_RELABEL = 256
F_NO_RELABEL = 512
F_CLAMP_CAS = 1024
F_PREFILTER = 2048
F_DEBUG_INVARIANTS = 4096
F_L2_PERSIST = 16384
F_LSA_EXCHANGE = 32768

K_NAMES = ["degree", "init", "rounds", "sum", "update", "peel", "validate", "relabel", "edgelist"]

STATUS = {0: "PICO_OK", 1: "PICO_EINVAL", 2: "PICO_ENOTSUP", 3: "PICO_ENOMEM",
          4: "PICO_ECUDA", 5: "PICO_ENCCL", 6: "PICO_EGRAPH"}


class PicoError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.msg = msg


class Stats(ctypes.Structure):
    """Mirror of pico_stats_t (include/pico.h)."""
    _fields_ = [
        ("rounds", ctypes.c_int64),
        ("levels", ctypes.c_int64),
        ("subrounds", ctypes.c_int64),
        ("kmax", ctypes.c_int64),
        ("frontier_total", ctypes.c_int64),
        ("init_slots_written", ctypes.c_int64),
        ("arcs_scanned", ctypes.c_int64),
        ("guarded_arcs", ctypes.c_int64),
        ("bins_read", ctypes.c_int64),
        ("pushes", ctypes.c_int64),
        ("alive_scanned", ctypes.c_int64),
        ("hub_fallbacks", ctypes.c_int64),
        ("segments", ctypes.c_int64),
        ("segments_init", ctypes.c_int64),
        ("kernel_count", ctypes.c_int64),
        ("pull_rounds", ctypes.c_int64),
        ("kernel_ms", ctypes.c_double * 9),
        ("kernel_launches", ctypes.c_int64 * 9),
        ("frontier_sizes", ctypes.POINTER(ctypes.c_int64)),
        ("frontier_sizes_cap", ctypes.c_int64),
        ("round_arcs", ctypes.POINTER(ctypes.c_int64)),
        ("round_ns", ctypes.POINTER(ctypes.c_int64)),
        ("algo", ctypes.c_int64),
        ("affected", ctypes.c_int64),
        ("bfs_levels", ctypes.c_int64),
        ("frontier_counts", ctypes.POINTER(ctypes.c_int32)),
        ("frontier_counts_cap", ctypes.c_int64),
    ]

    def to_dict(self) -> dict:
        d = {k: int(getattr(self, k)) for k, _ in self._fields_[:16]}
        d["algo"] = int(self.algo)
        d["affected"] = int(self.affected)
        d["bfs_levels"] = int(self.bfs_levels)
        d["kernel_ms"] = {K_NAMES[i]: float(self.kernel_ms[i]) for i in range(9) if self.kernel_launches[i]}
        d["kernel_launches"] = {K_NAMES[i]: int(self.kernel_launches[i]) for i in range(9) if self.kernel_launches[i]}
        return d


_lib = None


def header_functions() -> list[str]:
    """Every function declared in include/*.h (for the export test)."""
    names = []
    for fn in sorted(os.listdir(INCLUDE)):
        if not fn.endswith(".h"):
            continue
        txt = open(os.path.join(INCLUDE, fn)).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\**\s*(pico_[A-Za-z0-9_]+)\s*\(",
                             txt, flags=re.M):
            names.append(m.group(1))
    return sorted(set(names))


def load(path: str | None = None):
    """Load libpico.so (raises OSError if it is missing: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    p = path or os.environ.get("PICO_LIB") or LIB
    if not os.path.exists(p):
        raise OSError(f"libpico.so not built ({p}); run `python -m paper_2402_15253_b200.build` "
                      "or __graft_entry__.build()")
    lib = ctypes.CDLL(p)
    vp, i64, i32, u32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_uint32, ctypes.c_size_t
    lib.pico_coreness.argtypes = [vp, vp, i64, i64, i32, vp, vp]
    lib.pico_coreness.restype = i32
    lib.pico_workspace_bytes.argtypes = [i64, i64, i32, u32]
    lib.pico_workspace_bytes.restype = sz
    lib.pico_coreness_ex.argtypes = [vp, vp, i64, i64, i32, vp, vp, u32, vp, sz, ctypes.POINTER(Stats)]
    lib.pico_coreness_ex.restype = i32
    lib.pico_coreness_host.argtypes = [vp, vp, i64, i64, i32, vp, vp, u32, ctypes.POINTER(Stats)]
    lib.pico_coreness_host.restype = i32
    lib.pico_status_string.argtypes = [i32]
    lib.pico_status_string.restype = ctypes.c_char_p
    lib.pico_last_error.argtypes = []
    lib.pico_last_error.restype = ctypes.c_char_p
    lib.pico_version.argtypes = []
    lib.pico_version.restype = i32
    lib.pico_clamp_hammer.argtypes = [i32, ctypes.c_int32, ctypes.c_int32, i64, ctypes.POINTER(ctypes.c_int32),
                                      ctypes.POINTER(i64), ctypes.POINTER(i64), vp]
    lib.pico_clamp_hammer.restype = i32
    lib.pico_relabel_threshold.argtypes = []
    lib.pico_relabel_threshold.restype = i64
    _setup_shard(lib)
    lib.pico_dyn_create.argtypes = [vp, vp, i64, i64, u32, vp, ctypes.POINTER(Stats), ctypes.POINTER(vp)]
    lib.pico_dyn_create.restype = i32
    lib.pico_dyn_coreness.argtypes = [vp, vp]
    lib.pico_dyn_coreness.restype = i32
    lib.pico_dyn_delete_edges.argtypes = [vp, vp, vp, i64, ctypes.POINTER(Stats)]
    lib.pico_dyn_delete_edges.restype = i32
    lib.pico_dyn_insert_edges.argtypes = [vp, vp, vp, i64, ctypes.POINTER(Stats)]
    lib.pico_dyn_insert_edges.restype = i32
    lib.pico_dyn_destroy.argtypes = [vp]
    lib.pico_dyn_destroy.restype = i32
    _lib = lib
    return lib


def _setup_shard(lib):
    """Signatures of the sharded HistoCore / PeelOne entry points (include/pico_shard.h)."""
    if not hasattr(lib, "pico_shard_create"):
        return
    vp, i64, i32, u32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_uint32
    P64 = ctypes.POINTER(ctypes.c_int64)
    lib.pico_shard_create.argtypes = [vp, vp, i64, i64, i64, u32, vp, ctypes.POINTER(vp)]
    lib.pico_shard_create.restype = i32
    lib.pico_shard_degrees.argtypes = [vp, vp]
    lib.pico_shard_degrees.restype = i32
    lib.pico_shard_init.argtypes = [vp, vp, P64]
    lib.pico_shard_init.restype = i32
    lib.pico_shard_pack.argtypes = [vp, vp, i64, P64]
    lib.pico_shard_pack.restype = i32
    lib.pico_shard_apply.argtypes = [vp, vp, i64, P64]
    lib.pico_shard_apply.restype = i32
    lib.pico_shard_result.argtypes = [vp, vp]
    lib.pico_shard_result.restype = i32
    lib.pico_shard_destroy.argtypes = [vp]
    lib.pico_shard_destroy.restype = i32
    P32 = ctypes.POINTER(ctypes.c_int32)
    lib.pico_peel_shard_create.argtypes = [vp, vp, i64, i64, i64, u32, vp, ctypes.POINTER(vp), P32]
    lib.pico_peel_shard_create.restype = i32
    lib.pico_peel_shard_scan.argtypes = [vp, i32, vp, i64, P64, P32]
    lib.pico_peel_shard_scan.restype = i32
    lib.pico_peel_shard_apply.argtypes = [vp, vp, i64, vp, i64, P64, P32]
    lib.pico_peel_shard_apply.restype = i32
    lib.pico_peel_shard_result.argtypes = [vp, vp]
    lib.pico_peel_shard_result.restype = i32
    lib.pico_peel_shard_destroy.argtypes = [vp]
    lib.pico_peel_shard_destroy.restype = i32
    if hasattr(lib, "pico_coreness_sharded"):
        u8p = ctypes.POINTER(ctypes.c_uint8)
        lib.pico_comm_unique_id.argtypes = [u8p]
        lib.pico_comm_unique_id.restype = i32
        lib.pico_comm_init.argtypes = [i32, i32, u8p, ctypes.POINTER(vp)]
        lib.pico_comm_init.restype = i32
        lib.pico_comm_size.argtypes = [vp, ctypes.POINTER(i32), ctypes.POINTER(i32)]
        lib.pico_comm_size.restype = i32
        lib.pico_comm_destroy.argtypes = [vp]
        lib.pico_comm_destroy.restype = i32
        lib.pico_coreness_sharded.argtypes = [vp, vp, vp, i64, i64, i64, i64, i32, vp, vp]
        lib.pico_coreness_sharded.restype = i32
        lib.pico_coreness_sharded_ex.argtypes = [vp, vp, vp, i64, i64, i64, i64, i32, vp, vp, u32,
                                                 ctypes.POINTER(Stats)]
        lib.pico_coreness_sharded_ex.restype = i32


def check(rc: int):
    if rc != 0:
        raise PicoError(rc, load().pico_last_error().decode(errors="replace"))
