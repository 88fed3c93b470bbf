"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (plain pico_coreness_ex calls on the device CSR): the whole coreness
vector of every single-GPU config against the serial BZ oracle (SURVEY 8(c):
the result is unique, so the comparison is element by element), plus the
iteration counts the oracle pins cheaply at this size (k_max, PeelOne's
non-empty levels = number of distinct nonzero coreness values) and the
k-core definition check.  C2/C3 take seconds; T and C4 (2.1 G and 2.7 G arcs)
about a minute each of serial BZ on one host core."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


def _graph(cfg):
    import torch
    rp, ci = synth.CONFIGS[cfg].build(device=torch.device("cuda:0"))
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return rp, ci


def _check(cfg, kcore=True):
    import torch
    import paper_2402_15253_b200 as pico
    rp, ci = _graph(cfg)
    rp_np, ci_np = synth.to_numpy(rp, ci)
    ref = oracle.bz(rp_np, ci_np)
    nz = ref[ref > 0]
    for algo in ("histocore", "peelone"):
        st = pico.Stats()
        core = pico.coreness(rp, ci, algo=algo, stats=st).cpu().numpy()
        if not np.array_equal(core, ref):
            bad = np.flatnonzero(core != ref)
            raise AssertionError(f"{cfg} {algo}: {bad.size} mismatches, first v={bad[0]}: {core[bad[0]]} != {ref[bad[0]]}")
        if algo == "peelone":
            assert st.levels == np.unique(nz).size
            assert st.kmax == int(nz.max())
        else:
            assert st.rounds > 0
    if kcore:
        assert oracle.kcore_check(rp_np, ci_np, ref)
    del rp, ci
    torch.cuda.empty_cache()


@pytest.mark.parametrize("cfg", ["C2", "C3"])
def test_full_size_social(cfg):
    _check(cfg)


@pytest.mark.parametrize("cfg", ["T", "C4"])
def test_full_size_billion_edges(cfg):
    _check(cfg, kcore=False)


@pytest.mark.parametrize("parts", [2, 4])
def test_full_size_sharded_loopback(parts):
    """The sharded path (pull rounds over the rank edge lists and push rounds
    over the rank CSCs, gated per round) on the full C2 graph, P logical
    shards on one GPU, against the BZ oracle; l2 and every global |C_t| equal
    the single-GPU run's."""
    import torch
    import paper_2402_15253_b200 as pico
    from paper_2402_15253_b200 import sharded
    rp, ci = _graph("C2")
    ref = oracle.bz(*synth.to_numpy(rp, ci))
    core, rounds, sizes = sharded.coreness_loopback(rp, ci, parts)
    assert np.array_equal(core.cpu().numpy(), ref)
    st = pico.Stats()
    fs = np.zeros(1 << 12, dtype=np.int64)
    pico.coreness(rp, ci, stats=st, frontier_sizes=fs)
    assert rounds == st.rounds and sizes == [int(x) for x in fs[:st.rounds]]
    del rp, ci
    torch.cuda.empty_cache()


@pytest.mark.parametrize("parts", [2, 4])
def test_full_size_sharded_peel_loopback(parts):
    """Sharded PeelOne on the full C2 graph, P logical
    shards on one GPU, against the BZ oracle; non-empty levels, sub-rounds and
    k_max equal the single-GPU PeelOne's."""
    import torch
    import paper_2402_15253_b200 as pico
    from paper_2402_15253_b200 import sharded
    rp, ci = _graph("C2")
    ref = oracle.bz(*synth.to_numpy(rp, ci))
    run = sharded.coreness_loopback_peel(rp, ci, parts)
    assert np.array_equal(run.core_local.cpu().numpy(), ref)
    st = pico.Stats()
    pico.coreness(rp, ci, algo="peelone", stats=st)
    assert (run.levels, run.subrounds, run.kmax) == (st.levels, st.subrounds, st.kmax)
    del rp, ci
    torch.cuda.empty_cache()


@pytest.mark.parametrize("flags", [0, 32 | 128])
def test_full_size_frontier_sequence_c2(flags):
    """F_t = {v : h_t(v) != h_{t-1}(v)} of the synchronous Jacobi
    iteration, so l2 and EVERY |F_t| are pinned by oracle.jacobi_rounds --
    here on the full C2 graph in its default schedule (pull rounds over the
    edge list, push rounds, bench launch configuration) and with pull forced
    in every round over a many-bucket edge list (TINY_TILES | PULL_ALWAYS)."""
    import torch
    import paper_2402_15253_b200 as pico
    rp, ci = _graph("C2")
    rp_np, ci_np = synth.to_numpy(rp, ci)
    core_j, l2, sizes = oracle.jacobi_rounds(rp_np, ci_np)
    st = pico.Stats()
    fs = np.zeros(1 << 12, dtype=np.int64)
    core = pico.coreness(rp, ci, flags=flags, stats=st, frontier_sizes=fs).cpu().numpy()
    assert np.array_equal(core, core_j)
    assert st.rounds == l2
    assert [int(x) for x in fs[:l2]] == [int(x) for x in sizes]
    del rp, ci
    torch.cuda.empty_cache()
