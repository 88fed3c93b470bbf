"""Decremental HistoCore (include/pico_dyn.h): after
every batch of edge deletions the maintained coreness equals the BZ oracle's
coreness of the reduced graph, element by element, for the default schedule
and for forced pull rounds over a multi-bucket edge list (tombstones in both
the CSR copy and the edge list) and forced push rounds; a vertex that loses
every edge drops to coreness 0; a missing edge is rejected."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


def _edges(rp, ci):
    src = np.repeat(np.arange(rp.size - 1), np.diff(rp))
    keep = src < ci
    return np.stack([src[keep], ci[keep]], 1)


def _reduced(n, edges):
    rp, ci = synth.from_edge_list(n, [tuple(e) for e in edges.tolist()])
    return synth.to_numpy(rp, ci)


@pytest.mark.parametrize("cfg,flags", [("R12", 0), ("R12", 128 | 32), ("R12", 64), ("R14", 0)])
def test_decremental_batches(cfg, flags):
    import torch
    import paper_2402_15253_b200 as pico
    dev = torch.device("cuda:0")
    rp, ci = synth.to_numpy(*synth.CONFIGS[cfg].build())
    n = rp.size - 1
    edges = _edges(rp, ci)
    rng = np.random.default_rng(11)
    d = pico.DynamicCoreness(torch.from_numpy(rp).to(dev), torch.from_numpy(ci).to(dev), flags=flags)
    try:
        assert np.array_equal(d.coreness().cpu().numpy(), oracle.bz(rp, ci))
        # a hub loses every edge; then random batches of growing size
        hub = int(np.argmax(np.diff(rp)))
        batches = [np.flatnonzero((edges[:, 0] == hub) | (edges[:, 1] == hub))]
        alive = np.ones(len(edges), bool)
        alive[batches[0]] = False
        for size in (1, 17, len(edges) // 20, len(edges) // 5):
            idx = rng.choice(np.flatnonzero(alive), size=min(size, int(alive.sum())), replace=False)
            alive[idx] = False
            batches.append(idx)
        alive = np.ones(len(edges), bool)
        for b in batches:
            e = edges[b]
            d.delete_edges(torch.from_numpy(e[:, 0].astype(np.int32)), torch.from_numpy(e[:, 1].astype(np.int32)))
            alive[b] = False
            r_rp, r_ci = _reduced(n, edges[alive])
            ref = oracle.bz(r_rp, r_ci)
            got = d.coreness().cpu().numpy()
            assert np.array_equal(got, ref), (cfg, flags, int((got != ref).sum()))
        assert d.coreness()[hub].item() == 0
        # an edge that is no longer in the graph
        e = edges[batches[-1][:1]]
        with pytest.raises(pico.PicoError) as ei:
            d.delete_edges(torch.from_numpy(e[:, 0].astype(np.int32)), torch.from_numpy(e[:, 1].astype(np.int32)))
        assert ei.value.status == 1
    finally:
        d.close()


def test_decremental_duplicates_and_rejection():
    """A batch holding the same undirected edge twice and reversed is applied
    once (each arc claimed by one warp); a batch with a missing
    edge is rejected before anything changes and the handle stays usable."""
    import torch
    import paper_2402_15253_b200 as pico
    dev = torch.device("cuda:0")
    rp, ci = synth.to_numpy(*synth.CONFIGS["R12"].build())
    n = rp.size - 1
    edges = _edges(rp, ci)
    rng = np.random.default_rng(5)
    for flags in (0, 128 | 32):
        d = pico.DynamicCoreness(torch.from_numpy(rp).to(dev), torch.from_numpy(ci).to(dev), flags=flags)
        try:
            alive = np.ones(len(edges), bool)
            idx = rng.choice(len(edges), size=300, replace=False)
            e = edges[idx]
            # every edge three times: as given, reversed, as given again
            src = np.concatenate([e[:, 0], e[:, 1], e[:, 0]]).astype(np.int32)
            dst = np.concatenate([e[:, 1], e[:, 0], e[:, 1]]).astype(np.int32)
            perm = rng.permutation(src.size)
            d.delete_edges(torch.from_numpy(src[perm]), torch.from_numpy(dst[perm]))
            alive[idx] = False
            ref = oracle.bz(*_reduced(n, edges[alive]))
            assert np.array_equal(d.coreness().cpu().numpy(), ref)
            # one deleted edge among live ones: rejected, nothing applied
            live = np.flatnonzero(alive)[:50]
            bad = np.concatenate([edges[live], edges[idx[:1]]])
            with pytest.raises(pico.PicoError) as ei:
                d.delete_edges(torch.from_numpy(bad[:, 0].astype(np.int32)),
                               torch.from_numpy(bad[:, 1].astype(np.int32)))
            assert ei.value.status == 1
            assert np.array_equal(d.coreness().cpu().numpy(), ref)
            # a self loop / out-of-range id / length mismatch
            for s_, t_ in (([3], [3]), ([n], [0]), ([-1], [2])):
                with pytest.raises(pico.PicoError):
                    d.delete_edges(torch.tensor(s_, dtype=torch.int32), torch.tensor(t_, dtype=torch.int32))
            with pytest.raises(ValueError):
                d.delete_edges(torch.tensor([1, 2], dtype=torch.int32), torch.tensor([3], dtype=torch.int32))
            # still usable: the live edges go
            d.delete_edges(torch.from_numpy(edges[live][:, 0].astype(np.int32)),
                           torch.from_numpy(edges[live][:, 1].astype(np.int32)))
            alive[live] = False
            assert np.array_equal(d.coreness().cpu().numpy(), oracle.bz(*_reduced(n, edges[alive])))
        finally:
            d.close()


# ----------------------------------------------------------------- insertions
def _graph_from(n, edges):
    return _reduced(n, np.asarray(edges, dtype=np.int64).reshape(-1, 2))


@pytest.mark.parametrize("cfg,flags", [("R12", 0), ("R12", 128 | 32), ("R12", 64), ("R14", 0)])
def test_incremental_insertions(cfg, flags):
    """Insertions (pico_dyn_insert_edges; "inserted or removed"):
    start from a graph with a share of its edges held back, insert them in
    batches of growing size (single edges, edges between high-core vertices,
    edges to isolated vertices, random batches), interleaved with deletions;
    after every batch the coreness equals BZ on the current graph."""
    import torch
    import paper_2402_15253_b200 as pico
    dev = torch.device("cuda:0")
    rp, ci = synth.to_numpy(*synth.CONFIGS[cfg].build())
    n = rp.size - 1
    edges = _edges(rp, ci)
    rng = np.random.default_rng(23)
    held = rng.random(len(edges)) < 0.3
    cur = set(map(tuple, edges[~held].tolist()))
    pool = [tuple(e) for e in edges[held].tolist()]
    rng.shuffle(pool)
    r_rp, r_ci = _graph_from(n, sorted(cur))
    d = pico.DynamicCoreness(torch.from_numpy(r_rp).to(dev), torch.from_numpy(r_ci).to(dev), flags=flags)
    try:
        core = oracle.bz(r_rp, r_ci)
        assert np.array_equal(d.coreness().cpu().numpy(), core)
        iso = np.flatnonzero(np.diff(r_rp) == 0)
        hi = np.argsort(-core)[:40]
        extra = []
        if iso.size >= 2:
            extra.append([(int(iso[0]), int(iso[1])), (int(iso[0]), int(hi[0]))])  # new vertices join
        new_hi = [(int(min(a, b)), int(max(a, b))) for a in hi for b in hi if a < b and (min(a, b), max(a, b)) not in cur]
        extra.append(new_hi[:25])  # densify the top core: coreness rises there
        batches = [[pool.pop()], [pool.pop()]] + extra
        for size in (7, 60, len(pool) // 3):
            batches.append([pool.pop() for _ in range(min(size, len(pool)))])
        for i, b in enumerate(batches):
            b = [e for e in b if e not in cur]
            if not b:
                continue
            st = pico.Stats()
            e = np.asarray(b, dtype=np.int64)
            d.insert_edges(torch.from_numpy(e[:, 0].astype(np.int32)), torch.from_numpy(e[:, 1].astype(np.int32)),
                           stats=st)
            cur |= set(b)
            ref = oracle.bz(*_graph_from(n, sorted(cur)))
            got = d.coreness().cpu().numpy()
            assert np.array_equal(got, ref), (cfg, flags, i, int((got != ref).sum()))
            assert 0 < st.affected <= n
            if i == 3:  # a deletion batch in between: both directions on the same handle
                dl = sorted(cur)[:: max(1, len(cur) // 50)][:50]
                de = np.asarray(dl, dtype=np.int64)
                d.delete_edges(torch.from_numpy(de[:, 0].astype(np.int32)),
                               torch.from_numpy(de[:, 1].astype(np.int32)))
                cur -= set(dl)
                ref = oracle.bz(*_graph_from(n, sorted(cur)))
                assert np.array_equal(d.coreness().cpu().numpy(), ref)
    finally:
        d.close()


def test_insertion_rejection_and_duplicates():
    """An inserted edge that already exists, a self loop or an id out of range
    rejects the whole batch before anything changes; the same new edge given
    twice and reversed is inserted once."""
    import torch
    import paper_2402_15253_b200 as pico
    dev = torch.device("cuda:0")
    rp, ci = synth.to_numpy(*synth.CONFIGS["R12"].build())
    n = rp.size - 1
    edges = _edges(rp, ci)
    cur = set(map(tuple, edges.tolist()))
    d = pico.DynamicCoreness(torch.from_numpy(rp).to(dev), torch.from_numpy(ci).to(dev))
    try:
        ref0 = oracle.bz(rp, ci)
        rng = np.random.default_rng(3)
        new = []
        while len(new) < 40:
            a, b = sorted(map(int, rng.integers(0, n, 2)))
            if a != b and (a, b) not in cur and (a, b) not in new:
                new.append((a, b))
        t = lambda x: torch.from_numpy(np.asarray(x, dtype=np.int32))
        for bad in ([new[0], tuple(edges[0])], [new[0], (5, 5)], [new[0], (0, n)]):
            bad = np.asarray(bad)
            with pytest.raises(pico.PicoError) as ei:
                d.insert_edges(t(bad[:, 0]), t(bad[:, 1]))
            assert ei.value.status == 1
            assert np.array_equal(d.coreness().cpu().numpy(), ref0)
        e = np.asarray(new)
        src = np.concatenate([e[:, 0], e[:, 1], e[:, 0]])
        dst = np.concatenate([e[:, 1], e[:, 0], e[:, 1]])
        d.insert_edges(t(src), t(dst))
        cur |= set(new)
        assert np.array_equal(d.coreness().cpu().numpy(), oracle.bz(*_graph_from(n, sorted(cur))))
    finally:
        d.close()
