"""T2/T3: GPU parity.  The CUDA path (through the C ABI) against the CPU
oracle, element by element (bit-exact: coreness is integer and unique,
SURVEY 8(c)), plus iteration counts: HistoCore's l2 and every |F_t| equal the
synchronous Index2core sweeps; PeelOne's non-empty levels equal the number of
distinct nonzero coreness values and its k_max the maximum."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

ALGOS = ("histocore", "peelone")


def _pico():
    import paper_2402_15253_b200 as pico
    return pico


def _variants(algo):
    pico = _pico()
    base = [0, pico.F_HOST_LOOP, pico.F_TINY_TILES, pico.F_TINY_TILES | pico.F_HOST_LOOP, pico.F_STATS,
            pico.F_RELABEL, pico.F_RELABEL | pico.F_TINY_TILES | pico.F_STATS]
    if algo == "histocore":
        base += [pico.F_PUSH_ONLY, pico.F_PULL_ALWAYS, pico.F_PULL_ALWAYS | pico.F_TINY_TILES,
                 pico.F_PULL_ALWAYS | pico.F_HOST_LOOP, pico.F_PUSH_ONLY | pico.F_HOST_LOOP,
                 pico.F_PREFILTER, pico.F_PREFILTER | pico.F_TINY_TILES]
    if algo == "peelone":
        base += [pico.F_CLAMP_SUB, pico.F_CLAMP_SUB | pico.F_HOST_LOOP, pico.F_CLAMP_SUB | pico.F_TINY_TILES,
                 pico.F_CLAMP_CAS, pico.F_CLAMP_CAS | pico.F_HOST_LOOP, pico.F_CLAMP_CAS | pico.F_TINY_TILES]
    return base


def _run(rp_np, ci_np, algo, flags=0, fs_cap=1 << 16):
    import torch
    pico = _pico()
    dev = torch.device("cuda:0")
    rp = torch.from_numpy(rp_np).to(dev)
    ci = torch.from_numpy(ci_np).to(dev)
    st = pico.Stats()
    fs = np.zeros(fs_cap, dtype=np.int64)
    core = pico.coreness(rp, ci, algo=algo, flags=flags, stats=st, frontier_sizes=fs)
    torch.cuda.synchronize()
    return core.cpu().numpy(), st, fs


def _check(rp, ci, algo, flags, ref=None, jac=None):
    if ref is None:
        ref = oracle.bz(rp, ci)
    core, st, fs = _run(rp, ci, algo, flags)
    if not np.array_equal(core, ref):
        bad = np.flatnonzero(core != ref)
        raise AssertionError(f"{algo} flags={flags}: {bad.size} mismatches, first v={bad[0]} "
                             f"gpu={core[bad[0]]} ref={ref[bad[0]]}")
    if algo == "histocore":
        if jac is None:
            jac = oracle.jacobi_rounds(rp, ci)
        _, l2, sizes = jac
        assert st.rounds == l2, (st.rounds, l2)
        assert list(fs[:l2]) == sizes
    else:
        nz = ref[ref > 0]
        assert st.levels == len(np.unique(nz))
        assert st.kmax == (int(nz.max()) if nz.size else 0)
        # vertices processed per level sum to the non-isolated count
        assert int(fs[:st.levels].sum()) == nz.size
        # bulk-synchronous sub-rounds of the dynamic frontier equal the
        # level-synchronous reference's (deterministic under BSP draining)
        _, _, lv, sr = oracle.peel_levels(rp, ci)
        assert st.levels == lv and st.subrounds == sr, (st.subrounds, sr)
    return st


# ------------------------------------------------------------------ fixtures
def _fixture_graphs():
    from conftest import parse_small_fixtures, parse_g1, csr_np
    out = []
    g = parse_g1()
    edges = [tuple(int(x) for x in p.split("-")) for p in g["edges"].split()]
    out.append(("G1", csr_np(6, edges)))
    for fx in parse_small_fixtures():
        out.append((fx["name"], csr_np(fx["n"], fx["edges"])))
    out.append(("K20", csr_np(20, [(i, j) for i in range(20) for j in range(i + 1, 20)])))
    out.append(("K5_7", csr_np(12, [(i, 5 + j) for i in range(5) for j in range(7)])))
    out.append(("star200", csr_np(201, [(0, i) for i in range(1, 201)])))
    out.append(("single", csr_np(2, [(0, 1)])))
    return out


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("name,g", _fixture_graphs(), ids=[x[0] for x in _fixture_graphs()])
def test_fixtures(algo, name, g):
    rp, ci = g
    for fl in _variants(algo):
        _check(rp, ci, algo, fl)


def test_g1_paper_values():
    """G1: coreness [1,1,2,2,2,2]; HistoCore l2 = 1; PO-dyn 2
    levels = k_max; Fig 6 path: v5 5 -> 2 with no slot writes."""
    from conftest import parse_g1, csr_np
    g = parse_g1()
    edges = [tuple(int(x) for x in p.split("-")) for p in g["edges"].split()]
    rp, ci = csr_np(6, edges)
    core, st, _ = _run(rp, ci, "histocore", _pico().F_STATS)
    assert core.tolist() == [1, 1, 2, 2, 2, 2] and st.rounds == 1
    assert st.guarded_arcs == 0  # UpdateHisto: no neighbour has core > 2
    core, st, _ = _run(rp, ci, "peelone", _pico().F_STATS)
    assert core.tolist() == [1, 1, 2, 2, 2, 2] and st.levels == 2 and st.kmax == 2


# ------------------------------------------------------------------ corpus
def _corpus():
    out = []
    for i, (n, p) in enumerate([(30, 0.2), (100, 0.02), (100, 0.05), (150, 0.2), (200, 0.8),
                                (200, 0.05), (64, 0.5), (180, 0.1)]):
        out.append((f"er{i}", synth.to_numpy(*synth.erdos_renyi(n, p, seed=1000 + i))))
    for i, (n, e) in enumerate([(1000, 2.2), (3000, 2.5), (5000, 2.1)]):
        out.append((f"cl{i}", synth.to_numpy(*synth.chung_lu(n, 10.0, e, seed=2000 + i))))
    out.append(("R12", synth.to_numpy(*synth.CONFIGS["R12"].build())))
    out.append(("R14", synth.to_numpy(*synth.CONFIGS["R14"].build())))
    return out


_CORPUS = None


def corpus():
    global _CORPUS
    if _CORPUS is None:
        _CORPUS = _corpus()
    return _CORPUS


@pytest.mark.parametrize("algo", ALGOS)
def test_corpus_all_variants(algo):
    for name, (rp, ci) in corpus():
        ref = oracle.bz(rp, ci)
        jac = oracle.jacobi_rounds(rp, ci) if algo == "histocore" else None
        for fl in _variants(algo):
            _check(rp, ci, algo, fl, ref, jac)


@pytest.mark.parametrize("algo", ALGOS)
def test_schedule_robustness_repeat(algo):
    """5 repetitions give the identical result (atomics interleave
    differently every run)."""
    rp, ci = synth.to_numpy(*synth.CONFIGS["R14"].build())
    ref = oracle.bz(rp, ci)
    jac = oracle.jacobi_rounds(rp, ci)
    for _ in range(5):
        _check(rp, ci, algo, 0, ref, jac if algo == "histocore" else None)


def test_er_property_corpus_200():
    """S:463 corpus: 200 ER graphs n <= 200, p in {0.02, 0.05, 0.2, 0.8}."""
    ps = [0.02, 0.05, 0.2, 0.8]
    for i in range(200):
        n = 20 + (i * 37) % 181
        rp, ci = synth.to_numpy(*synth.erdos_renyi(n, ps[i % 4], seed=5000 + i))
        ref = oracle.bz(rp, ci)
        for algo in ALGOS:
            core, _, _ = _run(rp, ci, algo)
            assert np.array_equal(core, ref), (i, algo)


# ------------------------------------------------------------ larger graphs
def test_c1_rmat16_full():
    """configs[0]: RMAT scale-16 ef16 vs the oracle, both algorithms, with the
    invariants of the north star (core <= deg, k-core definition)."""
    rp, ci = synth.to_numpy(*synth.CONFIGS["C1"].build())
    ref = oracle.bz(rp, ci)
    jac = oracle.jacobi_rounds(rp, ci)
    for algo in ALGOS:
        for fl in (0, _pico().F_HOST_LOOP, _pico().F_STATS, _pico().F_RELABEL):
            _check(rp, ci, algo, fl, ref, jac)
    assert oracle.kcore_check(rp, ci, ref)


def test_gpu_generator_matches_cpu():
    """The shared generator is bit-identical on CPU and GPU (inputs of the
    oracle and of the CUDA path are the same graph)."""
    import torch
    a = synth.CONFIGS["R14"].build(device="cpu")
    b = synth.CONFIGS["R14"].build(device=torch.device("cuda:0"))
    assert torch.equal(a[0], b[0].cpu()) and torch.equal(a[1], b[1].cpu())
    c = synth.erdos_renyi(300, 0.05, seed=9, device="cpu")
    d = synth.erdos_renyi(300, 0.05, seed=9, device=torch.device("cuda:0"))
    assert torch.equal(c[1], d[1].cpu())


def test_unsorted_rows_pull_passes():
    """Rows in arbitrary order are allowed (include/pico.h): the pull passes
    need ascending rows, detect the unsorted input and run a single pass --
    same coreness and the same |F_t| sequence."""
    rp, ci = synth.to_numpy(*synth.CONFIGS["R12"].build())
    ref = oracle.bz(rp, ci)
    jac = oracle.jacobi_rounds(rp, ci)
    rng = np.random.default_rng(7)
    ci2 = ci.copy()
    for v in range(rp.size - 1):
        seg = ci2[rp[v]:rp[v + 1]]
        rng.shuffle(seg)
    pico = _pico()
    for fl in (pico.F_PULL_ALWAYS | pico.F_TINY_TILES, pico.F_PULL_ALWAYS, pico.F_TINY_TILES, 0):
        _check(rp, ci2, "histocore", fl, ref, jac)


def test_c1_pull_always_passes():
    """C1 with every round in the pull direction, single pass and (tiny
    tiles) three v-range passes."""
    rp, ci = synth.to_numpy(*synth.CONFIGS["C1"].build())
    ref = oracle.bz(rp, ci)
    jac = oracle.jacobi_rounds(rp, ci)
    pico = _pico()
    for fl in (pico.F_PULL_ALWAYS, pico.F_PULL_ALWAYS | pico.F_TINY_TILES,
               pico.F_PULL_ALWAYS | pico.F_TINY_TILES | pico.F_HOST_LOOP):
        _check(rp, ci, "histocore", fl, ref, jac)


def test_auto_algorithm():
    """PICO_ALGO_AUTO resolves by the degree skew and
    size -- HistoCore on the skewed C1, PeelOne on a flat ER graph -- and
    stays bit-exact; stats.algo reports the choice."""
    for (rp, ci), want in ((synth.to_numpy(*synth.CONFIGS["C1"].build()), 0),
                           (synth.to_numpy(*synth.erdos_renyi(400, 0.05, seed=77)), 1)):
        ref = oracle.bz(rp, ci)
        core, st, _ = _run(rp, ci, "auto")
        assert st.algo == want
        assert np.array_equal(core, ref)


@pytest.mark.parametrize("algo", ["cntcore", "nbrcore"])
def test_index2core_ablations(algo):
    """CntCore (Alg 5) and NbrCore: the same coreness and
    the same synchronous rounds (l2 and every |C_t|) as the Jacobi reference,
    on the fixtures, the small corpus, rows in arbitrary order and C1."""
    graphs = [g for _, g in _fixture_graphs()] + [g for _, g in corpus()]
    rp, ci = synth.to_numpy(*synth.CONFIGS["R12"].build())
    ci2 = ci.copy()
    rng = np.random.default_rng(3)
    for v in range(rp.size - 1):
        rng.shuffle(ci2[rp[v]:rp[v + 1]])
    graphs += [(rp, ci2), synth.to_numpy(*synth.CONFIGS["C1"].build())]
    for rp, ci in graphs:
        ref = oracle.bz(rp, ci)
        _, l2, sizes = oracle.jacobi_rounds(rp, ci)
        core, st, fs = _run(rp, ci, algo, pico_flags_stats())
        assert np.array_equal(core, ref)
        assert st.rounds == l2 and list(fs[:l2]) == sizes
        assert st.kmax == (int(ref.max()) if ref.size else 0)


def pico_flags_stats():
    return _pico().F_STATS


def test_long_path_many_rounds():
    """A path needs l2 = (n-1)//2 synchronous rounds (pinned on small paths
    against the Jacobi reference): far beyond the per-round records, still a
    valid input, for every Index2core algorithm and PeelOne."""
    for n in (5, 8, 31, 64):
        rp, ci = synth.to_numpy(*synth.path(n))
        assert oracle.jacobi_rounds(rp, ci)[1] == (n - 1) // 2
    n = 140_001
    rp, ci = synth.to_numpy(*synth.path(n))
    for algo in ("histocore", "peelone", "cntcore"):
        core, st, _ = _run(rp, ci, algo, 0, fs_cap=16)
        assert (core == 1).all()
        if algo != "peelone":
            assert st.rounds == (n - 1) // 2


def test_debug_invariants():
    """PICO_F_DEBUG_INVARIANTS re-counts every vertex's
    histogram against the final estimates and checks the h-index fixed point
    on the device, for the default, push-only, pull-always (multi-bucket) and
    host-loop schedules."""
    pico = _pico()
    graphs = [synth.to_numpy(*synth.CONFIGS[c].build()) for c in ("R12", "R14", "C1")]
    graphs += [g for _, g in _fixture_graphs()]
    for rp, ci in graphs:
        ref = oracle.bz(rp, ci)
        for fl in (0, pico.F_PUSH_ONLY, pico.F_PULL_ALWAYS | pico.F_TINY_TILES, pico.F_HOST_LOOP):
            core, _, _ = _run(rp, ci, "histocore", fl | pico.F_DEBUG_INVARIANTS)
            assert np.array_equal(core, ref)


def test_frontier_counts_fig3():
    """pico_stats_t.frontier_counts (PICO_F_STATS): the rounds in which each
    vertex is a frontier -- the paper's Fig 3 measure -- equal the
    oracle's synchronous sweeps vertex by vertex, in every schedule (push,
    pull, tiny tiles, host loop) and through the compaction (F_RELABEL maps the
    counts back to the original ids)."""
    pico = _pico()
    graphs = [("R12", synth.to_numpy(*synth.CONFIGS["R12"].build())),
              ("C1", synth.to_numpy(*synth.CONFIGS["C1"].build())),
              ("chung-lu", synth.to_numpy(*synth.chung_lu(3000, 8.0, 2.3, seed=5)))]
    for name, (rp, ci) in graphs:
        ref, l2, _, _ = oracle.frontier_counts(rp, ci)
        n = rp.size - 1
        for fl in (0, pico.F_PUSH_ONLY, pico.F_PULL_ALWAYS, pico.F_PULL_ALWAYS | pico.F_TINY_TILES,
                   pico.F_HOST_LOOP, pico.F_RELABEL, pico.F_RELABEL | pico.F_PULL_ALWAYS):
            import torch
            dev = torch.device("cuda:0")
            fc = np.full(n + 3, -7, dtype=np.int32)
            st = pico.Stats()
            core = pico.coreness(torch.from_numpy(rp).to(dev), torch.from_numpy(ci).to(dev), algo="histocore",
                                 flags=fl | pico.F_STATS, stats=st, frontier_counts=fc)
            torch.cuda.synchronize()
            assert st.rounds == l2, (name, fl)
            assert np.array_equal(fc[:n], ref), (name, fl, int(np.flatnonzero(fc[:n] != ref)[0]))
            assert np.array_equal(core.cpu().numpy(), oracle.bz(rp, ci))


def test_peelone_window_rule_regression(monkeypatch):
    """PeelOne's far-list rebuild must leave every vertex of the level in the
    near list: with a window rule of 1.5k + 16 a single rebuild whose far
    minimum landed above the new window lost 7-194 vertices per RMAT graph
    (DESIGN.md section 7).  The rebuild now repeats until the level fits the
    window; this graph (RMAT-20, edge factor 8, seed 3: 11 wrong values before
    the fix) must be bit-exact under that rule and the default one."""
    import torch
    pico = _pico()
    rp, ci = synth.rmat(20, 8, seed=3, compact=True)
    rp_np, ci_np = synth.to_numpy(rp, ci)
    ref = oracle.bz(rp_np, ci_np)
    dev = torch.device("cuda:0")
    rpd, cid = rp.to(dev), ci.to(dev)
    for rule in ("3/2+16", "2/1+16", "5/4+4"):
        monkeypatch.setenv("PICO_PO_WINDOW", rule)
        core = pico.coreness(rpd, cid, algo="peelone").cpu().numpy()
        assert np.array_equal(core, ref), (rule, int((core != ref).sum()))
