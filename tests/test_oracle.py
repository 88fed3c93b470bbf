"""T0/T1: pin the CPU oracle (oracle/) to things other than itself -- the
paper's worked example, closed forms, brute force, networkx, invariants.
CPU only."""
import itertools
import random

import numpy as np
import pytest

from conftest import csr_np, parse_g1, parse_small_fixtures, golden_path


def _edges_of(rowptr, colidx):
    out = []
    for v in range(len(rowptr) - 1):
        for e in range(rowptr[v], rowptr[v + 1]):
            if v < colidx[e]:
                out.append((v, int(colidx[e])))
    return out


# ---------------------------------------------------------------- G1
def test_g1_coreness_degrees(oracle_mod):
    g = parse_g1()
    n = int(g["n"])
    edges = [tuple(int(x) for x in p.split("-")) for p in g["edges"].split()]
    rp, ci = csr_np(n, edges)
    assert list(np.diff(rp)) == [int(x) for x in g["degree"].split()]
    expect = [int(x) for x in g["coreness"].split()]
    assert list(oracle_mod.bz(rp, ci)) == expect
    assert oracle_mod.brute_coreness(n, edges) == expect
    core, l2, fs = oracle_mod.jacobi_rounds(rp, ci)
    assert list(core) == expect and l2 == int(g["histocore_l2"])
    core, kmax, lv, sr = oracle_mod.peel_levels(rp, ci)
    assert list(core) == expect
    assert lv == int(g["peel_levels"]) and sr == int(g["peel_subrounds"]) and kmax == 2


def test_g1_fig6_histogram(oracle_mod):
    """Fig 6: v5's histogram over its neighbours' degrees is
    {1:{v0,v1}, 2:{v2,v4}, 3:{v3}} and its h-index is 2."""
    g = parse_g1()
    edges = [tuple(int(x) for x in p.split("-")) for p in g["edges"].split()]
    rp, ci = csr_np(6, edges)
    deg = np.diff(rp)
    vals = deg[ci[rp[5]:rp[6]]]
    hist = {}
    for x in vals:
        hist[int(x)] = hist.get(int(x), 0) + 1
    expect = dict((int(a), int(b)) for a, b in (p.split(":") for p in g["v5_histogram"].split()))
    assert hist == expect
    assert oracle_mod.hindex(vals) == int(g["v5_hindex"])
    # histogram_state with core = degrees at v5 (cap bin = deg 5 -> count >= 5 = 0)
    st = oracle_mod.histogram_state(rp, ci, deg, 5)
    assert st[1] == 2 and st[2] == 2 and st[3] == 1 and st[4] == 0 and st[5] == 0


# ------------------------------------------------------- small fixtures (S:*)
@pytest.mark.parametrize("fx", parse_small_fixtures(), ids=lambda f: f["name"])
def test_small_fixtures(oracle_mod, fx):
    rp, ci = csr_np(fx["n"], fx["edges"])
    assert list(oracle_mod.bz(rp, ci)) == fx["core"]
    assert oracle_mod.brute_coreness(fx["n"], fx["edges"]) == fx["core"]
    core, l2, _ = oracle_mod.jacobi_rounds(rp, ci)
    assert list(core) == fx["core"] and l2 == fx["l2"]
    core, kmax, lv, _ = oracle_mod.peel_levels(rp, ci)
    assert list(core) == fx["core"]
    assert lv == len(set(c for c in fx["core"] if c > 0))
    assert kmax == max(fx["core"] + [0])


# ------------------------------------------------------------- closed forms
@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 13])
def test_closed_forms(oracle_mod, n):
    # K_n -> n-1, P_n -> 1 (n>=2), C_n -> 2 (n>=3), star -> 1, edgeless -> 0
    kn = [(i, j) for i in range(n) for j in range(i + 1, n)]
    assert list(oracle_mod.bz(*csr_np(n, kn))) == [n - 1] * n
    pn = [(i, i + 1) for i in range(n - 1)]
    assert list(oracle_mod.bz(*csr_np(n, pn))) == ([1] * n if n >= 2 else [0])
    if n >= 3:
        cn = [(i, (i + 1) % n) for i in range(n)]
        assert list(oracle_mod.bz(*csr_np(n, cn))) == [2] * n
    st = [(0, i) for i in range(1, n + 1)]
    assert list(oracle_mod.bz(*csr_np(n + 1, st))) == [1] * (n + 1)
    assert list(oracle_mod.bz(*csr_np(n, []))) == [0] * n


@pytest.mark.parametrize("a,b", [(1, 1), (2, 3), (3, 3), (4, 7), (6, 2)])
def test_complete_bipartite(oracle_mod, a, b):
    e = [(i, a + j) for i in range(a) for j in range(b)]
    assert list(oracle_mod.bz(*csr_np(a + b, e))) == [min(a, b)] * (a + b)


def test_random_trees_are_1(oracle_mod):
    rng = random.Random(5)
    for _ in range(50):
        n = rng.randint(2, 60)
        e = [(i, rng.randrange(i)) for i in range(1, n)]
        assert list(oracle_mod.bz(*csr_np(n, e))) == [1] * n


def test_empty_graph(oracle_mod):
    rp = np.zeros(1, dtype=np.int64)
    ci = np.zeros(0, dtype=np.int32)
    assert oracle_mod.bz(rp, ci).size == 0
    assert oracle_mod.jacobi_rounds(rp, ci)[1] == 0


# ------------------------------------------------------------- brute force
def test_exhaustive_n_le_6(oracle_mod):
    """Every labelled simple graph on n <= 6 vertices: BZ == brute force,
    Jacobi fixed point == BZ, level peel == BZ."""
    for n in range(1, 7):
        pairs = [(i, j) for i in range(n) for j in range(i + 1, n)]
        for mask in range(1 << len(pairs)):
            e = [pairs[i] for i in range(len(pairs)) if mask >> i & 1]
            rp, ci = csr_np(n, e)
            b = oracle_mod.brute_coreness(n, e)
            assert list(oracle_mod.bz(rp, ci)) == b, (n, e)
            if mask % 7 == 0:
                assert list(oracle_mod.jacobi_rounds(rp, ci)[0]) == b
                assert list(oracle_mod.peel_levels(rp, ci)[0]) == b


def test_exhaustive_n_le_7_in_c(oracle_mod):
    """Every labelled simple graph on n <= 7 vertices (2^21 at n = 7): BZ ==
    the C brute force (oracle_brute, its own adjacency matrix, SURVEY 8(c)
    "brute force n <= 7 exhaustive")."""
    for n in range(1, 8):
        assert oracle_mod.exhaustive_mismatches(n) == 0, n


def test_brute_c_matches_python_brute(oracle_mod):
    """The C brute force is pinned to the pure-Python one on random
    graphs up to n = 40, so the exhaustive check above rests on it."""
    rng = random.Random(41)
    for _ in range(300):
        n = rng.randint(1, 40)
        pairs = [(i, j) for i in range(n) for j in range(i + 1, n)]
        p = rng.random() * 0.6
        e = [q for q in pairs if rng.random() < p]
        assert oracle_mod.brute_c(n, e) == oracle_mod.brute_coreness(n, e), (n, e)


def test_peel_subrounds_closed_forms(oracle_mod):
    """Level and BSP sub-round counts of the level-synchronous peel on graphs
    whose peel is known by hand: a path P_n peels one vertex from each end
    per sub-round (1 level, ceil(n/2) sub-rounds); a cycle and K_n go in one
    sub-round of one level; a star takes its leaves, then its centre (1
    level, 2 sub-rounds); disjoint unions add their levels' sub-rounds."""
    def run(n, e):
        rp, ci = csr_np(n, e)
        core, km, lv, sr = oracle_mod.peel_levels(rp, ci)
        assert list(core) == oracle_mod.brute_coreness(n, e)
        return lv, sr
    for n in range(2, 13):
        assert run(n, [(i, i + 1) for i in range(n - 1)]) == (1, (n + 1) // 2), n
    for n in range(3, 10):
        assert run(n, [(i, (i + 1) % n) for i in range(n)]) == (1, 1)
        assert run(n, [(i, j) for i in range(n) for j in range(i + 1, n)]) == (1, 1)
    for leaves in range(2, 9):
        assert run(leaves + 1, [(0, i) for i in range(1, leaves + 1)]) == (1, 2)
    # P5 + K4 (vertices 5..8): level 1 three sub-rounds, level 3 one
    e = [(i, i + 1) for i in range(4)] + [(5 + i, 5 + j) for i in range(4) for j in range(i + 1, 4)]
    assert run(9, e) == (2, 4)


def test_random_n7(oracle_mod):
    rng = random.Random(7)
    pairs = [(i, j) for i in range(7) for j in range(i + 1, 7)]
    for _ in range(3000):
        e = [p for p in pairs if rng.random() < rng.random()]
        rp, ci = csr_np(7, e)
        assert list(oracle_mod.bz(rp, ci)) == oracle_mod.brute_coreness(7, e)


def test_random_n_le_40(oracle_mod):
    rng = random.Random(40)
    for _ in range(400):
        n = rng.randint(2, 40)
        p = rng.choice([0.05, 0.1, 0.2, 0.4, 0.7])
        e = [(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < p]
        rp, ci = csr_np(n, e)
        b = oracle_mod.brute_coreness(n, e)
        assert list(oracle_mod.bz(rp, ci)) == b
        assert list(oracle_mod.jacobi_rounds(rp, ci)[0]) == b
        assert list(oracle_mod.peel_levels(rp, ci)[0]) == b


# ---------------------------------------------------------------- HINDEX
def test_hindex_golden(oracle_mod):
    with open(golden_path("hindex.txt")) as f:
        for line in f:
            if line.startswith("#") or "->" not in line:
                continue
            lhs, rhs = line.split("->")
            vals = [int(x) for x in lhs.split()]
            assert oracle_mod.hindex(vals) == int(rhs), line
            assert oracle_mod.hindex_sorted(vals) == int(rhs), line


def test_hindex_random_multisets(oracle_mod):
    """1000 random multisets (sizes 0-64, values 0-64) vs the
    sort-based textbook h-index and the two conditions of Alg 2 P:145-146."""
    rng = random.Random(1000)
    for _ in range(1000):
        vals = [rng.randint(0, 64) for _ in range(rng.randint(0, 64))]
        h = oracle_mod.hindex(vals)
        assert h == oracle_mod.hindex_sorted(vals)
        assert sum(x >= h for x in vals) >= h
        assert sum(x >= h + 1 for x in vals) <= h


# ------------------------------------------------------- Jacobi / l2 pins
def _py_jacobi(n, rp, ci, hfun):
    """Independent synchronous Index2core: every sweep recomputes every vertex
    from the previous sweep's values with a sort-based h-index."""
    cur = [int(rp[v + 1] - rp[v]) for v in range(n)]
    sizes = []
    while True:
        nxt = [hfun([cur[ci[e]] for e in range(rp[v], rp[v + 1])]) for v in range(n)]
        ch = sum(a != b for a, b in zip(cur, nxt))
        if ch == 0:
            return cur, sizes
        sizes.append(ch)
        cur = nxt


def test_jacobi_vs_python_sweeps(oracle_mod):
    rng = random.Random(77)
    for _ in range(150):
        n = rng.randint(2, 60)
        p = rng.choice([0.05, 0.1, 0.3, 0.6])
        e = [(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < p]
        rp, ci = csr_np(n, e)
        core, l2, fs = oracle_mod.jacobi_rounds(rp, ci)
        pc, psz = _py_jacobi(n, rp, ci, oracle_mod.hindex_sorted)
        assert list(core) == pc
        assert l2 == len(psz) and fs == psz


def _py_frontier_counts(n, rp, ci, hfun):
    """Independent Fig 3 measure: per-vertex frontier multiplicity
    and the (frontier, neighbour) pairs whose neighbour stays unchanged in the
    next sweep, from plain Python sweeps with the sort-based h-index."""
    cur = [int(rp[v + 1] - rp[v]) for v in range(n)]
    fc = [0] * n
    front = []
    un = tot = 0
    while True:
        nxt = [hfun([cur[ci[e]] for e in range(rp[v], rp[v + 1])]) for v in range(n)]
        for v in front:
            for e in range(rp[v], rp[v + 1]):
                tot += 1
                un += nxt[ci[e]] == cur[ci[e]]
        front = [v for v in range(n) if nxt[v] != cur[v]]
        if not front:
            return fc, un, tot
        for v in front:
            fc[v] += 1
        cur = nxt


def test_frontier_counts_vs_python(oracle_mod):
    """oracle_frontier_counts (the Fig 3 measure) against an independent
    Python sweep on 150 random graphs; its sum is the sum of the pinned |F_t|
    of oracle_jacobi_rounds and its l2 the same."""
    rng = random.Random(78)
    for _ in range(150):
        n = rng.randint(2, 60)
        p = rng.choice([0.05, 0.1, 0.3, 0.6])
        e = [(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < p]
        rp, ci = csr_np(n, e)
        fc, l2, un, tot = oracle_mod.frontier_counts(rp, ci)
        pfc, pun, ptot = _py_frontier_counts(n, rp, ci, oracle_mod.hindex_sorted)
        assert list(fc) == pfc and (un, tot) == (pun, ptot)
        _, jl2, fs = oracle_mod.jacobi_rounds(rp, ci)
        assert l2 == jl2 and int(fc.sum()) == sum(fs)


def test_frontier_counts_closed_forms(oracle_mod):
    """Closed forms: a star K_1,k (k >= 2) changes only its centre, once (deg
    k -> 1); K_n never changes; P5 = 0-1-2-3-4 changes 1 and 3 in sweep 1
    (h-index of {1, 2} = 1) and 2 in sweep 2 (neighbours now {1, 1}); of the
    sweep-1 frontier's neighbour pairs (1: {0, 2}, 3: {2, 4}) only those to 2
    see a change in sweep 2.  G1 (l2 = 1): the frontier is {v : h1 < deg}."""
    from conftest import parse_g1
    for k in (2, 3, 7):
        rp, ci = csr_np(k + 1, [(0, i) for i in range(1, k + 1)])
        fc, l2, un, tot = oracle_mod.frontier_counts(rp, ci)
        assert list(fc) == [1] + [0] * k and l2 == 1
        assert tot == k and un == k  # the leaves' estimates stay 1
    rp, ci = csr_np(5, [(i, j) for i in range(5) for j in range(i + 1, 5)])
    fc, l2, un, tot = oracle_mod.frontier_counts(rp, ci)
    assert list(fc) == [0] * 5 and l2 == 0 and tot == 0
    rp, ci = csr_np(5, [(0, 1), (1, 2), (2, 3), (3, 4)])
    fc, l2, un, tot = oracle_mod.frontier_counts(rp, ci)
    assert list(fc) == [0, 1, 1, 1, 0] and l2 == 2
    # sweep-1 frontier {1, 3}: pairs (1,0) (1,2) (3,2) (3,4); in sweep 2 only 2 changes;
    # sweep-2 frontier {2}: pairs (2,1) (2,3), unchanged in the (empty) sweep 3
    assert tot == 6 and un == 4
    g = parse_g1()
    edges = [tuple(int(x) for x in p.split("-")) for p in g["edges"].split()]
    n = 1 + max(max(e) for e in edges)
    rp, ci = csr_np(n, edges)
    fc, l2, _, _ = oracle_mod.frontier_counts(rp, ci)
    deg = np.diff(rp)
    h1 = [oracle_mod.hindex([int(deg[u]) for u in ci[rp[v]:rp[v + 1]]]) for v in range(n)]
    assert l2 == 1 and list(fc) == [int(h1[v] < deg[v]) for v in range(n)]


def test_jacobi_fixed_point_and_monotone(oracle_mod):
    """Fixed point HINDEX(core(nbr v)) == core(v); estimates only
    decrease so every |F_t| <= n."""
    import synth
    rp, ci = synth.to_numpy(*synth.CONFIGS["R12"].build())
    core, l2, fs = oracle_mod.jacobi_rounds(rp, ci)
    assert np.array_equal(core, oracle_mod.bz(rp, ci))
    n = rp.size - 1
    for v in range(0, n, 7):
        nb = core[ci[rp[v]:rp[v + 1]]]
        assert oracle_mod.hindex(nb) == core[v]
    assert l2 == len(fs) and all(0 < x <= n for x in fs)


# ------------------------------------------------ invariants + networkx
def _corpus():
    import synth
    out = []
    for i, (n, p) in enumerate([(50, 0.05), (120, 0.02), (200, 0.05), (150, 0.2), (80, 0.8)]):
        out.append((f"er{i}", synth.to_numpy(*synth.erdos_renyi(n, p, seed=1000 + i))))
    for i, n in enumerate([500, 2000]):
        out.append((f"cl{i}", synth.to_numpy(*synth.chung_lu(n, 8.0, 2.3, seed=2000 + i))))
    out.append(("R12", synth.to_numpy(*synth.CONFIGS["R12"].build())))
    out.append(("R14", synth.to_numpy(*synth.CONFIGS["R14"].build())))
    return out


@pytest.mark.parametrize("name,g", _corpus(), ids=[c[0] for c in _corpus()])
def test_bz_vs_networkx_and_invariants(oracle_mod, name, g):
    nx = pytest.importorskip("networkx")
    rp, ci = g
    n = rp.size - 1
    core = oracle_mod.bz(rp, ci)
    G = nx.Graph()
    G.add_nodes_from(range(n))
    G.add_edges_from(_edges_of(rp, ci))
    ref = nx.core_number(G)
    assert all(core[v] == ref[v] for v in range(n))
    deg = np.diff(rp)
    assert np.all(core <= deg) and np.all((core == 0) == (deg == 0))
    assert oracle_mod.kcore_check(rp, ci, core)
    # peel-level oracle agrees, its level count is #distinct nonzero coreness
    pc, kmax, lv, sr = oracle_mod.peel_levels(rp, ci)
    assert np.array_equal(pc, core) and kmax == core.max(initial=0)
    assert lv == len(set(core[core > 0].tolist())) and sr >= lv


def test_kcore_check_rejects_wrong(oracle_mod):
    """The definition check catches an over-estimate (a plausible mistake)."""
    rp, ci = csr_np(5, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3), (3, 4)])
    good = oracle_mod.bz(rp, ci)
    assert oracle_mod.kcore_check(rp, ci, good)
    bad = good.copy()
    bad[4] = 2  # pendant cannot be in a 2-core
    assert not oracle_mod.kcore_check(rp, ci, bad)


@pytest.mark.slow
def test_c1_vs_networkx(oracle_mod):
    """configs[0] (RMAT-16): BZ equals networkx.core_number."""
    nx = pytest.importorskip("networkx")
    import synth
    rp, ci = synth.to_numpy(*synth.CONFIGS["C1"].build())
    core = oracle_mod.bz(rp, ci)
    n = rp.size - 1
    G = nx.Graph()
    G.add_nodes_from(range(n))
    src = np.repeat(np.arange(n), np.diff(rp))
    m = src < ci
    G.add_edges_from(zip(src[m].tolist(), ci[m].tolist()))
    ref = nx.core_number(G)
    assert all(core[v] == ref[v] for v in range(n))
