import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: slower CPU test (still part of -m 'not gpu')")


def golden_path(name: str) -> str:
    return os.path.join(ROOT, "tests", "golden", name)


def parse_small_fixtures():
    """tests/golden/small_fixtures.txt -> list of dicts."""
    out = []
    with open(golden_path("small_fixtures.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            name, n, edges, core, l2, src = [x.strip() for x in line.split("|")]
            e = [tuple(int(t) for t in p.split("-")) for p in edges.split()] if edges else []
            out.append(dict(name=name, n=int(n), edges=e, core=[int(x) for x in core.split()],
                            l2=int(l2), src=src))
    return out


def parse_g1():
    d = {}
    with open(golden_path("g1.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            k, _, v = line.partition(" ")
            d[k] = v
    return d


def csr_np(n, edges):
    """Tiny numpy CSR builder for test fixtures (symmetric, dedup, sorted)."""
    import numpy as np
    s = set()
    for u, v in edges:
        if u != v:
            s.add((u, v))
            s.add((v, u))
    arcs = sorted(s)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    for u, _ in arcs:
        rowptr[u + 1] += 1
    rowptr = np.cumsum(rowptr).astype(np.int64)
    colidx = np.array([v for _, v in arcs], dtype=np.int32)
    return rowptr, colidx


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    oracle.build_oracle()
    return oracle
