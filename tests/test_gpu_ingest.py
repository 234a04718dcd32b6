"""Pipelined host-CSR ingest (kb_graph_create, kb_ingest.cu build_graph).

The columns arrive in chunks of whole rows, highest rows first; each chunk is
validated, copied into the slack layout, written into its SELL slots and its
lower arcs dropped into the symmetry buckets while the next chunk uploads.
Checked here against the oracle and a numpy restatement of
Graph.is_symmetric (graph.py:168-175), at chunk sizes from one row to the
whole graph, from pageable and from page-locked host memory.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import katz_oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_1807_03847_b200")
from paper_1807_03847_b200 import _lib  # noqa: E402

DEFAULT_CHUNK = 1 << 25


@pytest.fixture
def chunk():
    L = _lib.lib()

    def set_(arcs):
        _lib.check(L.kb_tune(b"ingest.chunk_arcs", int(arcs)))

    yield set_
    set_(DEFAULT_CHUNK)


def sym_np(ip, ix):
    """The arc set equals its reversal."""
    n = ip.size - 1
    src = np.repeat(np.arange(n, dtype=np.int64), np.diff(ip))
    fwd = np.sort(src * n + ix)
    rev = np.sort(ix.astype(np.int64) * n + src)
    return bool(np.array_equal(fwd, rev))


def csr_from_arcs(n, arcs):
    arcs = np.unique(np.asarray(arcs, dtype=np.int64).reshape(-1, 2), axis=0)
    ip = np.zeros(n + 1, dtype=np.int64)
    np.add.at(ip, arcs[:, 0] + 1, 1)
    return np.cumsum(ip), arcs[:, 1].astype(np.int32)


def device_sym(ip, ix):
    dg = P.DeviceGraph(ip, ix)
    try:
        return dg.is_symmetric()
    finally:
        dg.close()


@pytest.mark.parametrize("arcs", [7, 1000, 1 << 25])
def test_chunked_ingest_matches_oracle(chunk, arcs):
    chunk(arcs)
    g0 = O.rmat_graph(1 << 12, edge_factor=16, seed=5)
    dg = P.DeviceGraph(g0.indptr, g0.indices, split_threshold=64)
    assert dg.is_symmetric()
    ip = np.empty_like(g0.indptr)
    ix = np.empty_like(g0.indices)
    _lib.check(_lib.lib().kb_graph_get_csr(dg.handle, _lib.ptr(ip), _lib.ptr(ix)))
    np.testing.assert_array_equal(ip, g0.indptr)
    np.testing.assert_array_equal(ix, g0.indices)
    dg.close()
    # the SELL slots drive K1: the certified run equals the oracle's
    g = P.Graph.from_csr(g0.node_count, g0.indptr, g0.indices)
    st = P.init(g, P.Criterion.top_k(30, 1e-9), undirected=True)
    res = P.run(st, g)
    ores = O.run(O.OracleState(g0, O.Crit("topk", 1e-9, k=30)), g0)
    assert res.iterations_used == ores.iterations_used
    np.testing.assert_array_equal(res.order, ores.order)
    np.testing.assert_allclose(res.lower, ores.lower, rtol=1e-12, atol=0)
    np.testing.assert_allclose(res.upper, ores.upper, rtol=1e-12, atol=0)


@pytest.mark.parametrize("arcs", [1, 50, 1 << 25])
def test_symmetry_flag_at_ingest(chunk, arcs):
    chunk(arcs)
    rng = np.random.default_rng(11)
    n = 300
    e = rng.integers(0, n, size=(2000, 2))
    e = e[e[:, 0] != e[:, 1]]
    both = np.concatenate([e, e[:, ::-1]])
    ip, ix = csr_from_arcs(n, both)
    assert sym_np(ip, ix) and device_sym(ip, ix)
    # self-loops are their own reversal
    loops = np.stack([np.arange(0, n, 7)] * 2, axis=1)
    ip2, ix2 = csr_from_arcs(n, np.concatenate([both, loops]))
    assert device_sym(ip2, ix2)
    # drop one arc of a pair, in turn from the lower and the upper triangle
    for k in (0, 1, 17, len(e) - 1):
        u, v = e[k]
        keep = ~(((both[:, 0] == u) & (both[:, 1] == v)))
        ip3, ix3 = csr_from_arcs(n, both[keep])
        assert not sym_np(ip3, ix3)
        assert not device_sym(ip3, ix3)
    # equal per-row counts, different sets: 0->2, 1->0, 2->1
    ip4, ix4 = csr_from_arcs(3, [(0, 2), (1, 0), (2, 1)])
    assert not device_sym(ip4, ix4)
    # a directed chain and the empty graph
    ip5, ix5 = csr_from_arcs(5, [(0, 1), (1, 2)])
    assert not device_sym(ip5, ix5)
    assert device_sym(np.zeros(4, dtype=np.int64), np.zeros(0, dtype=np.int32))


def test_symmetry_random_asymmetric_many_chunks(chunk):
    chunk(64)
    rng = np.random.default_rng(3)
    n = 5000
    for trial in range(4):
        e = rng.integers(0, n, size=(30000, 2))
        e = e[e[:, 0] != e[:, 1]]
        both = np.concatenate([e, e[:, ::-1]])
        # perturb: flip some arcs' targets so a few reversals go missing
        m = trial * 3
        if m:
            idx = rng.choice(both.shape[0], size=m, replace=False)
            both[idx, 1] = (both[idx, 1] + 1) % n
            both = both[both[:, 0] != both[:, 1]]
        ip, ix = csr_from_arcs(n, both)
        assert device_sym(ip, ix) == sym_np(ip, ix)


def test_long_rows_and_hubs(chunk):
    # a star with a hub row longer than the per-block threshold (256 arcs) and the item size (2048)
    chunk(500)
    n = 4000
    hub = [(0, v) for v in range(1, n)] + [(v, 0) for v in range(1, n)]
    ip, ix = csr_from_arcs(n, hub)
    assert device_sym(ip, ix)
    ip2, ix2 = csr_from_arcs(n, hub[:-1])
    assert not device_sym(ip2, ix2)
    ip3, ix3 = csr_from_arcs(n, hub[1:])
    assert not device_sym(ip3, ix3)


@pytest.mark.parametrize("bad", ["unsorted", "duplicate", "range", "negative"])
def test_invalid_rows_rejected(chunk, bad):
    chunk(3)
    ip, ix = csr_from_arcs(6, [(0, 1), (0, 3), (1, 0), (2, 4), (2, 5), (3, 0), (4, 2),
                               (5, 2)])
    ix = ix.copy()
    if bad == "unsorted":
        ix[0], ix[1] = ix[1], ix[0]
    elif bad == "duplicate":
        ix[4] = ix[3]
    elif bad == "range":
        ix[2] = 6
    else:
        ix[5] = -1
    with pytest.raises(P.ParameterError, match="strictly ascending"):
        P.DeviceGraph(ip, ix)


def test_pinned_host_arrays(chunk):
    """Page-locked arrays take the path that queues every chunk up front."""
    chunk(2000)
    L = _lib.lib()
    g0 = O.rmat_graph(1 << 11, edge_factor=8, seed=9)
    ip, ix = np.ascontiguousarray(g0.indptr), np.ascontiguousarray(g0.indices)
    for a in (ip, ix):
        _lib.check(L.kb_host_register(_lib.ptr(a), a.nbytes))
    try:
        dg = P.DeviceGraph(ip, ix)
        assert dg.is_symmetric()
        ip2 = np.empty_like(ip)
        ix2 = np.empty_like(ix)
        _lib.check(L.kb_graph_get_csr(dg.handle, _lib.ptr(ip2), _lib.ptr(ix2)))
        np.testing.assert_array_equal(ip2, ip)
        np.testing.assert_array_equal(ix2, ix)
        dg.close()
    finally:
        for a in (ip, ix):
            L.kb_host_unregister(_lib.ptr(a))


@pytest.mark.parametrize("arcs", [1, 1 << 25])
def test_degenerate_graphs(chunk, arcs):
    """No rows, one row, rows that are all empty, self-loops only, and a
    long run of empty rows between chunk boundaries."""
    chunk(arcs)
    assert device_sym(np.zeros(1, dtype=np.int64), np.zeros(0, dtype=np.int32))
    assert device_sym(np.zeros(2, dtype=np.int64), np.zeros(0, dtype=np.int32))
    ip, ix = csr_from_arcs(5, [(v, v) for v in range(5)])
    assert device_sym(ip, ix)
    ip, ix = csr_from_arcs(1000, [(0, 999), (999, 0), (1, 998)])
    assert not device_sym(ip, ix)
    ip, ix = csr_from_arcs(1000, [(0, 999), (999, 0), (1, 998), (998, 1)])
    assert device_sym(ip, ix)
    # a run on it: the two edges rank first, every other node has bound 0
    g = P.Graph.from_csr(1000, ip, ix)
    res = P.run(P.init(g, P.Criterion.top_k(4, 1e-9), undirected=True), g)
    assert sorted(res.top(4)) == [0, 1, 998, 999]


def test_init_symmetry_from_the_device_copy_on_large_graphs():
    """Above 4M arcs init takes the symmetry test from the ingest's device
    result instead of sorting every arc key on the host; the verdict (and
    the error for an asymmetric arc set) is the same."""
    g0 = O.rmat_graph(1 << 18, edge_factor=16, seed=4)
    assert g0.indptr[-1] > (1 << 22)
    g = P.Graph.from_csr(g0.node_count, g0.indptr, g0.indices)
    st = P.init(g, P.Criterion.top_k(10, 1e-6), undirected=True)
    assert st.r == 0
    ix = g0.indices.copy()
    ip = g0.indptr
    # drop one arc u -> v (keep v -> u): the arc set is no longer symmetric
    u = int(np.argmax(np.diff(ip)))
    keep = np.ones(ix.size, dtype=bool)
    keep[ip[u]] = False
    ip2 = ip.copy()
    ip2[u + 1:] -= 1
    gd = P.Graph.from_csr(g0.node_count, ip2, ix[keep])
    assert not gd.is_symmetric()
    with pytest.raises(P.ParameterError, match="symmetric"):
        P.init(gd, P.Criterion.top_k(10, 1e-6), undirected=True)
