"""Dynamic updates (K4) on the device vs the reference's golden sequences,
a fresh static recompute, and the reference suite's behavioural rules
(pkg/tests/test_dynamic.py restated)."""
from __future__ import annotations

import random

import numpy as np
import pytest

from oracle import katz_oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_1807_03847_b200")

REL = 1e-12


def fresh_to_depth(g, st):
    """Static state on g's current arcs, iterated to st.r (test_dynamic.py:18-24)."""
    other = P.init(g, st.criterion, alpha=st.alpha, undirected=st.undirected,
                   max_iterations=max(st.r, 1))
    for _ in range(st.r):
        P.iterate_once(other, g)
    return other


def assert_state_matches(st, fresh, rel=REL):
    assert len(st.levels) == len(fresh.levels)
    for mine, theirs in zip(st.levels, fresh.levels):
        np.testing.assert_allclose(mine, theirs, rtol=rel, atol=rel)
    np.testing.assert_allclose(st.katz, fresh.katz, rtol=rel, atol=rel)
    np.testing.assert_allclose(st.lower, fresh.lower, rtol=rel, atol=rel)
    np.testing.assert_allclose(st.upper, fresh.upper, rtol=rel, atol=rel)


def er(n, p, seed, undirected=True):
    rng = random.Random(seed)
    e = []
    for i in range(n):
        for j in range(i + 1 if undirected else 0, n):
            if i != j and rng.random() < p:
                e.append((i, j))
    return P.Graph.from_edges(n, e, undirected=undirected)


def random_batch(g, rng, max_ops=5, undirected=False):
    n = g.node_count
    present = list(g.arcs())
    if undirected:
        present = [(u, v) for u, v in present if u < v]
    rng.shuffle(present)
    dels = present[:rng.randint(0, min(max_ops, len(present)))]
    ins = []
    want = rng.randint(0, max_ops)
    tries = 0
    while len(ins) < want and tries < 50 * max_ops:
        tries += 1
        u, v = rng.randrange(n), rng.randrange(n)
        if u == v or g.has_arc(u, v) or (u, v) in ins:
            continue
        if undirected:
            u, v = min(u, v), max(u, v)
            if (u, v) in ins:
                continue
        ins.append((u, v))
    if undirected:
        dels = [a for uv in dels for a in (uv, uv[::-1])]
        ins = [a for uv in ins for a in (uv, uv[::-1])]
    return P.EdgeBatch(insertions=ins, deletions=dels)


def test_golden_dynamic_sequences(golden_index, dynamic_cases):
    """The reference's own update sequences: states within 1e-12 of its
    delta-propagated values, bit-identical to a fresh static recompute, and
    the same UpdateStats."""
    for c in golden_index["dynamic"]:
        name = c["name"]
        g = P.Graph.from_edges(c["n"], dynamic_cases[f"{name}/edges0"])
        kind = c["kind"]
        crit = {"ranking": P.Criterion.ranking(c["epsilon"]),
                "score": P.Criterion.score(c["epsilon"]),
                "topk": P.Criterion.top_k(c["k"] or 1, c["epsilon"])}[kind]
        st = P.init(g, crit, alpha=c["alpha"], undirected=c["undirected"])
        P.run(st, g)
        for i, step in enumerate(c["steps"]):
            p = f"{name}/b{i}"
            batch = P.EdgeBatch(insertions=[tuple(x) for x in dynamic_cases[p + "/ins"].tolist()],
                                deletions=[tuple(x) for x in dynamic_cases[p + "/del"].tolist()])
            P.update_batch(st, g, batch, theta=c["theta"])
            assert st.r == step["r"], p
            np.testing.assert_allclose(st.katz, dynamic_cases[p + "/katz"], rtol=REL, atol=1e-13)
            np.testing.assert_allclose(st.lower, dynamic_cases[p + "/lower"], rtol=REL, atol=1e-13)
            np.testing.assert_allclose(st.upper, dynamic_cases[p + "/upper"], rtol=REL, atol=1e-13)
            fresh = fresh_to_depth(g, st)
            np.testing.assert_array_equal(st.katz, fresh.katz, err_msg=p)
            np.testing.assert_array_equal(st.lower, fresh.lower, err_msg=p)
            np.testing.assert_array_equal(st.upper, fresh.upper, err_msg=p)
            s = st.last_update_stats
            assert s.seeds == step["seeds"], p
            assert s.aborted_level == step["aborted_level"], p
            assert s.level_sizes == step["level_sizes"], p
            assert s.visited == step["visited"], p
            assert s.reactivated == step["reactivated"], p
            assert s.resumed_iterations == step["resumed_iterations"], p
            assert st.gamma == step["gamma"], p


def test_single_insertion_and_deletion_match_fresh():
    g = P.Graph.from_edges(6, [(i, i + 1) for i in range(5)], undirected=True)
    st = P.init(g, P.Criterion.ranking(1e-8), alpha=0.2, undirected=True)
    P.run(st, g)
    P.update_batch(st, g, P.EdgeBatch(insertions=[(0, 3), (3, 0)]), theta=1.0)
    assert_state_matches(st, fresh_to_depth(g, st))
    g2 = P.Graph.from_edges(8, [(i, (i + 1) % 8) for i in range(8)], undirected=True)
    st2 = P.init(g2, P.Criterion.ranking(1e-8), alpha=0.2, undirected=True)
    P.run(st2, g2)
    P.update_batch(st2, g2, P.EdgeBatch(deletions=[(2, 3), (3, 2)]), theta=1.0)
    assert_state_matches(st2, fresh_to_depth(g2, st2))


def test_directed_mixed_and_random_streams():
    g = er(40, 0.08, 13, undirected=False)
    st = P.init(g, P.Criterion.score(1e-9), alpha=0.05)
    P.run(st, g)
    rng = random.Random(99)
    P.update_batch(st, g, random_batch(g, rng, max_ops=6), theta=1.0)
    assert_state_matches(st, fresh_to_depth(g, st))
    rng = random.Random(7)
    g = er(35, 0.1, 2)
    st = P.init(g, P.Criterion.ranking(1e-7), alpha=0.02, undirected=True)
    P.run(st, g)
    for _ in range(8):
        P.update_batch(st, g, random_batch(g, rng, max_ops=4, undirected=True), theta=1.0)
        assert_state_matches(st, fresh_to_depth(g, st))
        assert P.check_converged(st)


def test_theta_zero_forces_full_recompute_and_routes_agree():
    g = P.Graph.from_edges(12, [(i, (i + 1) % 12) for i in range(12)], undirected=True)
    st = P.init(g, P.Criterion.score(1e-8), alpha=0.2, undirected=True)
    P.run(st, g)
    P.update_batch(st, g, P.EdgeBatch(insertions=[(0, 6), (6, 0)]), theta=0.0)
    s = st.last_update_stats
    assert s.aborted_level == 1 and s.level_sizes == []
    assert_state_matches(st, fresh_to_depth(g, st))
    g1, g2 = er(30, 0.1, 5), er(30, 0.1, 5)
    ins = [(0, 17), (17, 0)] if not g1.has_arc(0, 17) else next(
        [(u, v), (v, u)] for u in range(30) for v in range(u + 1, 30) if not g1.has_arc(u, v))
    dele = next([(u, v), (v, u)] for u, v in sorted(g1.arcs()) if u < v and (u, v) != ins[0])
    b = P.EdgeBatch(insertions=ins, deletions=dele)
    s1 = P.init(g1, P.Criterion.score(1e-9), alpha=0.05, undirected=True)
    s2 = P.init(g2, P.Criterion.score(1e-9), alpha=0.05, undirected=True)
    P.run(s1, g1)
    P.run(s2, g2)
    P.update_batch(s1, g1, b, theta=1.0)
    P.update_batch(s2, g2, b, theta=0.0)
    assert s1.last_update_stats.aborted_level is None
    assert s2.last_update_stats.aborted_level == 1
    np.testing.assert_array_equal(s1.katz, s2.katz)
    np.testing.assert_array_equal(s1.lower, s2.lower)
    np.testing.assert_array_equal(s1.upper, s2.upper)


def test_insert_then_delete_restores_levels():
    e = []
    for r in range(5):
        for c in range(5):
            v = r * 5 + c
            if c + 1 < 5:
                e.append((v, v + 1))
            if r + 1 < 5:
                e.append((v, v + 5))
    g = P.Graph.from_edges(25, e, undirected=True)
    st = P.init(g, P.Criterion.score(1e-9), alpha=0.1, undirected=True)
    P.run(st, g)
    levels0 = [lvl.copy() for lvl in st.levels]
    arc = [(0, 6), (6, 0)]
    P.update_batch(st, g, P.EdgeBatch(insertions=arc), theta=1.0)
    P.update_batch(st, g, P.EdgeBatch(deletions=arc), theta=1.0)
    assert len(st.levels) >= len(levels0)
    for mine, orig in zip(st.levels, levels0):
        np.testing.assert_allclose(mine, orig, rtol=1e-12, atol=1e-14)
    assert_state_matches(st, fresh_to_depth(g, st))


def test_empty_batch_is_a_noop():
    g = P.Graph.from_edges(10, [(0, i) for i in range(1, 10)], undirected=True)
    st = P.init(g, P.Criterion.top_k(3, 1e-7), undirected=True)
    P.run(st, g)
    lo, up = st.lower.copy(), st.upper.copy()
    P.update_batch(st, g, P.EdgeBatch())
    np.testing.assert_array_equal(st.lower, lo)
    np.testing.assert_array_equal(st.upper, up)
    assert P.check_converged(st)


def test_guards():
    g = P.Graph.from_edges(4, [(0, 1), (1, 2), (2, 3)], undirected=True)
    st = P.init(g, P.Criterion.ranking(1e-6), undirected=True)
    P.run(st, g)
    arcs_before = set(g.arcs())
    with pytest.raises(P.ParameterError):   # alpha admission before mutation
        P.update_batch(st, g, P.EdgeBatch(insertions=[(1, 3), (3, 1)]))
    assert set(g.arcs()) == arcs_before and P.check_converged(st)
    c6 = lambda: P.Graph.from_edges(6, [(i, (i + 1) % 6) for i in range(6)], undirected=True)
    g = c6()
    st = P.init(g, P.Criterion.ranking(1e-6), alpha=0.2, undirected=True)
    P.run(st, g)
    with pytest.raises(P.ParameterError):
        P.update_batch(st, g, P.EdgeBatch(insertions=[(0, 3)]))
    with pytest.raises(P.ParameterError):
        P.update_batch(st, g, P.EdgeBatch(), theta=1.5)
    with pytest.raises(P.BatchPreconditionError):
        P.update_batch(st, g, P.EdgeBatch(deletions=[(0, 3), (3, 0)]))
    g.insert_arcs([(0, 3), (3, 0)])
    with pytest.raises(P.StateError):
        P.update_batch(st, g, P.EdgeBatch())
    g = c6()
    st = P.init(g, P.Criterion.ranking(1e-6), alpha=0.2, undirected=True, keep_all_levels=False)
    P.run(st, g)
    with pytest.raises(P.StateError):
        P.update_batch(st, g, P.EdgeBatch())


def test_topk_reactivates_displaced_nodes():
    edges = [(0, i) for i in range(1, 12)] + [(12, 13), (13, 14), (12, 14)]
    g = P.Graph.from_edges(15, edges, undirected=True)
    st = P.init(g, P.Criterion.top_k(2, 1e-6), alpha=0.05, undirected=True)
    P.run(st, g)
    assert st.active.size < 15
    dels = []
    for leaf in range(4, 12):
        dels += [(0, leaf), (leaf, 0)]
    P.update_batch(st, g, P.EdgeBatch(deletions=dels), theta=1.0)
    assert st.last_update_stats.reactivated > 0
    assert P.check_converged(st)
    fresh = P.init(g, P.Criterion.top_k(2, 1e-6), alpha=0.05, undirected=True)
    assert P.ranking_result(st).top(2) == P.run(fresh, g).top(2)


def test_locality_and_level_growth():
    e = [(i, i + 1) for i in range(29)]
    g = P.Graph.from_edges(30, e, undirected=True)
    st = P.init(g, P.Criterion.score(0.5), alpha=0.3, undirected=True)
    P.run(st, g)
    P.update_batch(st, g, P.EdgeBatch(deletions=[(10, 11), (11, 10)]), theta=1.0)
    sizes = st.last_update_stats.level_sizes
    assert sizes[0] == 2
    for a, b in zip(sizes, sizes[1:]):
        assert b - a <= 2


@pytest.mark.parametrize("nb", [100, 1000])
def test_rmat_s16_batches_match_static_recompute(nb):
    """C5 in miniature: insertion batches on R-MAT s16 ef16 vs a static run
    on the post-batch graph (same r, order, top-100; bounds 1e-12)."""
    g0 = O.rmat_graph(65536, edge_factor=16, seed=42)
    g = P.Graph.from_csr(g0.node_count, g0.indptr, g0.indices)
    st = P.init(g, P.Criterion.top_k(100, 1e-6), undirected=True)
    P.run(st, g)
    deg = np.diff(g0.indptr)
    dmax = int(deg.max())
    rng = np.random.default_rng(7)
    ins = set()
    while len(ins) < nb:
        u, v = (int(x) for x in rng.integers(0, 65536, 2))
        if u == v:
            continue
        u, v = min(u, v), max(u, v)
        if (u, v) in ins or g.has_arc(u, v) or deg[u] + 1 >= dmax or deg[v] + 1 >= dmax:
            continue
        ins.add((u, v))
    arcs = [a for uv in sorted(ins) for a in (uv, uv[::-1])]
    P.update_batch(st, g, P.EdgeBatch(insertions=arcs))
    res = P.ranking_result(st)
    assert P.check_converged(st)
    same_depth = fresh_to_depth(g, st)
    np.testing.assert_allclose(st.lower, same_depth.lower, rtol=REL, atol=0)
    np.testing.assert_allclose(st.upper, same_depth.upper, rtol=REL, atol=0)
    fres = P.run(P.init(g, P.Criterion.top_k(100, 1e-6), undirected=True), g)
    assert res.top(100) == fres.top(100)
    # the oracle on the post-batch arcs agrees on the certified top-100
    ip, ix = g.csr_arrays()
    og = O.CSRGraph(65536, ip, ix, symmetric=True)
    ores = O.run(O.OracleState(og, O.Crit("topk", 1e-6, k=100)), og)
    assert ores.top(100) == fres.top(100)


@pytest.mark.parametrize("heavy_dense", [0, 10**9])
def test_heavy_row_repair_routes_bitwise(heavy_dense):
    """Heavy rows (> split arcs) of a sparse level are re-folded from their
    SELL segments -- per row (k_heavy_rows_fold) or all at once through K1
    (run_segments + k_heavy_finish); both give a fresh static run's bits.
    The batch also edits heavy rows (patched in place)."""
    from paper_1807_03847_b200 import _lib
    L = _lib.lib()
    _lib.check(L.kb_tune(b"dyn.heavy_dense", heavy_dense))
    try:
        g0 = O.rmat_graph(65536, edge_factor=16, seed=42)
        g = P.Graph.from_csr(g0.node_count, g0.indptr, g0.indices)
        st = P.init(g, P.Criterion.top_k(100, 1e-6), undirected=True)
        P.run(st, g)
        deg = np.diff(g0.indptr)
        heavy = np.nonzero((deg > 2048) & (deg + 1 < deg.max()))[0]
        assert heavy.size > 0
        rng = np.random.default_rng(11)
        ins = set()
        for h in heavy[:8]:               # edit some heavy rows directly
            while True:
                v = int(rng.integers(0, 65536))
                if v != h and not g.has_arc(int(h), v) and deg[v] + 1 < deg.max():
                    ins.add((min(int(h), v), max(int(h), v)))
                    break
        while len(ins) < 600:
            u, v = (int(x) for x in rng.integers(0, 65536, 2))
            if u == v or g.has_arc(u, v) or max(deg[u], deg[v]) + 1 >= deg.max():
                continue
            ins.add((min(u, v), max(u, v)))
        arcs = [a for uv in sorted(ins) for a in (uv, uv[::-1])]
        P.update_batch(st, g, P.EdgeBatch(insertions=arcs))
        fresh = fresh_to_depth(g, st)
        for mine, theirs in zip(st.levels, fresh.levels):
            np.testing.assert_array_equal(mine, theirs)
        np.testing.assert_array_equal(st.lower, fresh.lower)
        np.testing.assert_array_equal(st.upper, fresh.upper)
        # one more K1 pass after the repair: the dense heavy route's segment
        # pass must leave the K1 work counter in a state K1 resets (it once
        # kept a converged check's "already zeroed" mark, so this pass
        # skipped rows)
        P.iterate_once(st, g)
        fresh = fresh_to_depth(g, st)
        np.testing.assert_array_equal(st.levels[-1], fresh.levels[-1])
        np.testing.assert_array_equal(st.lower, fresh.lower)
    finally:
        _lib.check(L.kb_tune(b"dyn.heavy_dense", 256))


@pytest.mark.parametrize("seed", [5, 6, 7])
def test_heavy_segment_pass_then_full_level_k1(seed):
    """A converged check pre-zeroes K1's work counter; a dense heavy repair
    (run_segments) at a local level then takes work from it, and the next
    dense level runs K1 over every row.  That K1 must start from a reset
    counter (it once skipped the reset and left rows unvisited): the levels
    stay bit-identical to a fresh static run.  A few arcs between low-degree
    nodes next to hubs put hubs in a local level."""
    from paper_1807_03847_b200 import _lib
    L = _lib.lib()
    _lib.check(L.kb_tune(b"dyn.heavy_dense", 0))
    try:
        g0 = O.rmat_graph(65536, edge_factor=16, seed=42)
        g = P.Graph.from_csr(g0.node_count, g0.indptr, g0.indices)
        st = P.init(g, P.Criterion.top_k(100, 1e-6), undirected=True)
        P.run(st, g)
        deg = np.diff(g0.indptr)
        hub = deg > 2048
        cand = [u for u in np.nonzero((deg >= 1) & (deg <= 3))[0]
                if hub[g0.indices[g0.indptr[u]:g0.indptr[u + 1]]].any()]
        rng = np.random.default_rng(seed)
        rng.shuffle(cand)
        ins = set()
        for a, b in zip(cand[0:24:2], cand[1:24:2]):
            if not g.has_arc(int(a), int(b)):
                ins.add((min(int(a), int(b)), max(int(a), int(b))))
        ins = sorted(ins)
        # two batches: the first update's closing check is what leaves the
        # counter pre-zeroed (P.run ends on a speculative K1 instead)
        for part in (ins[:len(ins) // 2], ins[len(ins) // 2:]):
            arcs = [a for uv in part for a in (uv, uv[::-1])]
            P.update_batch(st, g, P.EdgeBatch(insertions=arcs))
        fresh = fresh_to_depth(g, st)
        assert len(st.levels) == len(fresh.levels)
        for mine, theirs in zip(st.levels, fresh.levels):
            np.testing.assert_array_equal(mine, theirs)
        np.testing.assert_array_equal(st.lower, fresh.lower)
        np.testing.assert_array_equal(st.upper, fresh.upper)
    finally:
        _lib.check(L.kb_tune(b"dyn.heavy_dense", 256))


@pytest.mark.parametrize("nb", [100, 1000, 10000])
def test_rmat_s16_updates_match_oracle_update_batch(nb):
    """C5's rule pinned against the oracle's update_batch (dynamic.py:126-211
    restated; tests/test_oracle.py pins it to the reference's own golden
    sequences): on R-MAT s16 ef16 with 1e2 / 1e3 / 1e4-edge insertion
    batches, UpdateStats are identical field by field (level sizes, abort
    level, visited, reactivated, resumed iterations) and the bounds agree
    within 1e-12 (the reference's delta pushes vs the device's pull
    recompute).  The batch comes in as an (m, 2) int64 array."""
    n = 65536
    g0 = O.rmat_graph(n, edge_factor=16, seed=42)
    g = P.Graph.from_csr(n, g0.indptr, g0.indices)
    crit = P.Criterion.top_k(100, 1e-6)
    st = P.init(g, crit, undirected=True)
    P.run(st, g)
    deg = np.diff(g0.indptr)
    dmax = int(deg.max())
    rng = np.random.default_rng(7 + nb)
    cand = rng.integers(0, n, size=(4 * nb, 2))
    cand = np.sort(cand[cand[:, 0] != cand[:, 1]], axis=1)
    cand = np.unique(cand, axis=0)
    cand = cand[(deg[cand[:, 0]] + 1 < dmax) & (deg[cand[:, 1]] + 1 < dmax)]
    cand = cand[~g._has_keys(cand[:, 0] * n + cand[:, 1])]
    e = cand[rng.permutation(cand.shape[0])[:nb]]
    arcs = np.concatenate([e, e[:, ::-1]])
    P.update_batch(st, g, P.EdgeBatch(insertions=arcs))
    stats = st.last_update_stats
    og = O.AdjGraph.from_csr(g0)
    ost = O.OracleState(og, O.Crit("topk", 1e-6, k=100))
    O.run(ost, og)
    ostats = O.update_batch(ost, og, [tuple(x) for x in arcs.tolist()], [])
    for f in ("batch_size", "seeds", "visited", "level_sizes", "reactivated",
              "aborted_level", "resumed_iterations"):
        assert getattr(stats, f) == getattr(ostats, f), f
    assert st.r == ost.r
    np.testing.assert_allclose(st.lower, ost.lower, rtol=REL, atol=0)
    np.testing.assert_allclose(st.upper, ost.upper, rtol=REL, atol=0)
    assert P.ranking_result(st).top(100) == O.ranking_result(ost).top(100)


@pytest.mark.parametrize("split", [100, 2048])
def test_long_overflow_rows_bitwise(split):
    """Rows edited past their SELL lane are recomputed after K1 from the
    canonical CSR; those longer than 256 arcs by a block each (k_ovf_long:
    staged gathers, one serial chain, split-sized segments combined in
    order, segment boundaries falling inside the 2048-value chunks when
    split = 100).  Levels and bounds equal a fresh static layout's with the
    same split bit for bit, after the update and after one more K1."""
    from paper_1807_03847_b200 import generators as G
    from paper_1807_03847_b200.engine import DeviceGraph
    g = G.rmat_graph(65536, edge_factor=16, seed=42, split_threshold=split)
    crit = P.Criterion.top_k(100, 1e-6)
    st = P.init(g, crit, undirected=True)
    P.run(st, g)
    deg = g.out_degrees()
    rng = np.random.default_rng(3)
    long_rows = np.nonzero((deg > 300) & (deg + 40 < deg.max()))[0]
    assert long_rows.size > 20
    ins = set()
    for u in long_rows[:60]:
        k = 0
        while k < 24:                      # enough to outgrow any lane
            v = int(rng.integers(0, 65536))
            if v != u and deg[v] + 30 < deg.max() and not g.has_arc(int(u), v):
                ins.add((min(int(u), v), max(int(u), v)))
                k += 1
    e = np.array(sorted(ins), dtype=np.int64)
    P.update_batch(st, g, P.EdgeBatch(insertions=np.concatenate([e, e[:, ::-1]])))
    info = g.device_graph.info()
    assert info.overflow_long > 0, (info.overflow_rows, info.overflow_long)
    ip, ix = g.csr_arrays()
    fg = G.DeviceResidentGraph(DeviceGraph(ip, ix, split_threshold=split))
    fresh = fresh_to_depth(fg, st)
    for mine, theirs in zip(st.levels, fresh.levels):
        np.testing.assert_array_equal(mine, theirs)
    np.testing.assert_array_equal(st.lower, fresh.lower)
    np.testing.assert_array_equal(st.upper, fresh.upper)
    P.iterate_once(st, g)
    P.iterate_once(fresh, fg)
    np.testing.assert_array_equal(st.levels[-1], fresh.levels[-1])
    np.testing.assert_array_equal(st.lower, fresh.lower)


def test_mixed_batches_relocate_and_respread(capfd, monkeypatch):
    """The device-side batch path end to end: edits grouped by row on the
    device, rows that outgrow their slack relocated to the tail, then (tail
    room made small with kb_tune dyn.tail_room) the tail exhausted and the
    layout re-spread, with deletions of earlier insertions mixed in.  After
    every batch the device arcs are exactly the expected set and the levels
    and bounds equal a fresh static layout's bit for bit."""
    from paper_1807_03847_b200 import _lib
    from paper_1807_03847_b200 import generators as G
    L = _lib.lib()
    _lib.check(L.kb_tune(b"dyn.tail_room", 0))
    try:
        n = 4096
        g = G.rmat_graph(n, edge_factor=8, seed=3)
        crit = P.Criterion.top_k(20, 1e-6)
        st = P.init(g, crit, undirected=True, alpha=1e-5, max_iterations=400)
        P.run(st, g)
        ip, ix = g.csr_arrays()
        present = set(zip(np.repeat(np.arange(n), np.diff(ip)).tolist(), ix.tolist()))
        rng = np.random.default_rng(5)
        inserted = []
        monkeypatch.setenv("KB_TRACE", "1")
        for _ in range(6):
            hubs = rng.choice(n, 24, replace=False)       # rows that grow fast
            ins = set()
            while len(ins) < 1500:
                u = int(hubs[rng.integers(0, 24)]) if rng.random() < 0.6 else int(rng.integers(0, n))
                v = int(rng.integers(0, n))
                a = (min(u, v), max(u, v))
                if u == v or a in ins or a in present:
                    continue
                ins.add(a)
            dels, inserted = inserted[:500], inserted[500:]
            ia = np.array(sorted(ins), dtype=np.int64)
            da = np.array(dels, dtype=np.int64).reshape(-1, 2)
            P.update_batch(st, g, P.EdgeBatch(insertions=np.concatenate([ia, ia[:, ::-1]]),
                                              deletions=np.concatenate([da, da[:, ::-1]])))
            for u, v in dels:
                present.discard((u, v))
                present.discard((v, u))
            for u, v in ins:
                present.add((u, v))
                present.add((v, u))
            inserted += sorted(ins)
            ip, ix = g.csr_arrays()
            got = set(zip(np.repeat(np.arange(n), np.diff(ip)).tolist(), ix.tolist()))
            assert got == present
            fresh = fresh_to_depth(P.Graph.from_csr(n, ip, ix), st)
            for mine, theirs in zip(st.levels, fresh.levels):
                np.testing.assert_array_equal(mine, theirs)
            np.testing.assert_array_equal(st.lower, fresh.lower)
            np.testing.assert_array_equal(st.upper, fresh.upper)
        err = capfd.readouterr().err
        assert "relocate rows" in err and "respread" in err, err[-2000:]
    finally:
        _lib.check(L.kb_tune(b"dyn.tail_room", 1 << 20))


def test_grid_updates_through_the_narrow_kernel_bitwise():
    """An all-narrow graph (a grid) runs K1 as the TMA-staged narrow kernel,
    also in the level repair (level-only launches, no katz stream) and with
    the RANKING chain's fused pair test.  Insert and delete a few grid-local
    arcs, keeping every degree <= 4: levels and bounds equal a fresh static
    layout's bit for bit, and the ranking equals a fresh run's."""
    from paper_1807_03847_b200 import generators as G
    side = 96
    n = side * side
    g = G.grid_graph(n)
    crit = P.Criterion.ranking(1e-9)
    st = P.init(g, crit, undirected=True, max_iterations=400)
    P.run(st, g)
    deg = g.out_degrees()
    rng = np.random.default_rng(2)
    ins, dele = set(), set()
    ip, ix = g.csr_arrays()
    for _ in range(400):
        u = int(rng.integers(0, n))
        if deg[u] >= 4:
            continue
        for v in (u + 2, u + 2 * side):       # a short grid-local chord
            if v < n and deg[v] < 4 and not g.has_arc(u, v) and (u, v) not in ins:
                ins.add((u, v))
                deg[u] += 1
                deg[v] += 1
                break
        if len(ins) >= 30:
            break
    for u in range(0, n, 997):                # a few deletions of existing arcs
        nb = ix[ip[u]:ip[u + 1]]
        if nb.size:
            v = int(nb[0])
            dele.add((min(u, v), max(u, v)))
    ia = np.array(sorted(ins), dtype=np.int64).reshape(-1, 2)
    da = np.array(sorted(dele), dtype=np.int64).reshape(-1, 2)
    P.update_batch(st, g, P.EdgeBatch(insertions=np.concatenate([ia, ia[:, ::-1]]),
                                      deletions=np.concatenate([da, da[:, ::-1]])))
    ip, ix = g.csr_arrays()
    fg = P.Graph.from_csr(n, ip, ix)
    fresh = fresh_to_depth(fg, st)
    for mine, theirs in zip(st.levels, fresh.levels):
        np.testing.assert_array_equal(mine, theirs)
    np.testing.assert_array_equal(st.lower, fresh.lower)
    np.testing.assert_array_equal(st.upper, fresh.upper)
    res = P.ranking_result(st)
    fres = P.run(P.init(fg, crit, undirected=True, alpha=st.alpha, max_iterations=400), fg)
    np.testing.assert_array_equal(res.order, fres.order)
