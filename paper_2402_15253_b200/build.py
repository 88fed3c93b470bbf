"""Build libpico.so (the C-ABI library, include/pico.h) in-tree with nvcc for
sm_100a.  No torch extension: the library has a plain C ABI; Python reaches it
through ctypes (paper_2402_15253_b200/_lib.py)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libpico.so")

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC",
    "-Xcompiler", "-fvisibility=default",
]
LINK_FLAGS = [
    "-shared",
    "-ldl",  # NCCL is loaded with dlopen by the sharded entry points
]


def nccl_device_include() -> str | None:
    """Include directory of an NCCL >= 2.28 with the device API headers
    (nccl_device.h), e.g. the nvidia-nccl wheel torch depends on; None if
    absent (lsa_exchange.cu then builds its stub)."""
    cands = [os.environ.get("PICO_NCCL_INCLUDE")]
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
        if spec and spec.submodule_search_locations:
            cands += [os.path.join(p, "include") for p in spec.submodule_search_locations]
    except (ImportError, ValueError):
        pass
    cands += glob.glob(os.path.join(sys.prefix, "lib", "python3*", "site-packages", "nvidia", "nccl", "include"))
    for c in cands:
        if c and os.path.exists(os.path.join(c, "nccl_device.h")):
            return c
    return None


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
                              + glob.glob(os.path.join(INCLUDE, "*.h")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in deps())


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Compile every csrc/*.cu to an object in parallel (one nvcc per file),
    then link the shared library."""
    import tempfile
    from concurrent.futures import ThreadPoolExecutor
    target = out or LIB
    if not force and out is None and not needs_build():
        return LIB
    tmp = target + f".tmp{os.getpid()}"
    with tempfile.TemporaryDirectory(prefix="pico_build_") as d:
        def compile_one(src):
            obj = os.path.join(d, os.path.basename(src) + ".o")
            extra = []
            if os.path.basename(src) == "lsa_exchange.cu":
                inc = nccl_device_include()
                extra = ["-I" + inc, "-DPICO_HAVE_NCCL_DEVICE=1"] if inc else ["-DPICO_HAVE_NCCL_DEVICE=0"]
            cmd = ([nvcc()] + NVCC_FLAGS + ["-D" + x for x in defines] + extra
                   + ["-I" + INCLUDE, "-I" + CSRC, "-c", src, "-o", obj])
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            subprocess.check_call(cmd)
            return obj
        srcs = sources()
        with ThreadPoolExecutor(max(1, min(len(srcs), os.cpu_count() or 1))) as ex:
            objs = list(ex.map(compile_one, srcs))
        cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a"] + LINK_FLAGS + ["-o", tmp] + objs
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
