"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for PICO (arXiv 2402.15253).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  The product path
(``paper_2402_15253_b200``) never imports it and shares no code with it.

* :mod:`oracle.coreness` -- ctypes bindings to ``oracle.c`` (BZ bucket peel,
  HINDEX, synchronous Index2core sweeps, level-synchronous peel, k-core check)
  plus pure-Python brute force for tiny graphs.

Parity status of every function is in the header of ``oracle.c`` and in
DESIGN.md ("Oracle and its pins").  None is "parity unpinned".
"""
from .coreness import (  # noqa: F401
    build_oracle,
    bz,
    hindex,
    jacobi_rounds,
    frontier_counts,
    peel_levels,
    kcore_check,
    brute_coreness,
    hindex_sorted,
    histogram_state,
    brute_c,
    exhaustive_mismatches,
)
