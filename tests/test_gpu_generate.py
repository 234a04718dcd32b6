"""Device generators and the device-resident graph surface (B200)."""
from __future__ import annotations

import hashlib

import numpy as np
import pytest

from oracle import katz_oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_1807_03847_b200")
from paper_1807_03847_b200 import generators as G  # noqa: E402


def h16(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


@pytest.mark.parametrize("ef", [8, 16])
def test_device_rmat_is_the_reference_generator(golden_index, ef):
    d = golden_index["digests"][f"rmat_s16_ef{ef}_csr"]
    g = G.rmat_graph(65536, edge_factor=ef, seed=42)
    ip, ix = g.csr_arrays()
    assert g.arc_count == d["nnz"] and g.max_out_degree() == d["dmax"]
    assert h16(ip) == d["indptr"] and h16(ix) == d["indices"]
    assert g.is_symmetric()


@pytest.mark.parametrize("n", [1, 2, 7, 1000, 65536])
def test_device_grid_is_the_reference_generator(n):
    g = G.grid_graph(n)
    ip, ix = g.csr_arrays()
    o = O.grid_graph(n)
    np.testing.assert_array_equal(ip, o.indptr)
    np.testing.assert_array_equal(ix, o.indices)


def test_rmat_s20_matches_oracle_generator():
    g = G.rmat_graph(1 << 20, edge_factor=16, seed=42)
    o = O.rmat_graph(1 << 20, edge_factor=16, seed=42)
    ip, ix = g.csr_arrays()
    assert g.arc_count == 31400214
    np.testing.assert_array_equal(ip, o.indptr)
    np.testing.assert_array_equal(ix, o.indices)


def test_device_resident_graph_dynamic_matches_host_graph():
    gd = G.rmat_graph(4096, edge_factor=16, seed=3)
    ip, ix = gd.csr_arrays()
    gh = P.Graph.from_csr(4096, ip.copy(), ix.copy())
    sd = P.init(gd, P.Criterion.top_k(50, 1e-9), undirected=True)
    sh = P.init(gh, P.Criterion.top_k(50, 1e-9), undirected=True)
    P.run(sd, gd)
    P.run(sh, gh)
    rng = np.random.default_rng(1)
    deg = np.diff(ip)
    for _ in range(3):
        ins = set()
        while len(ins) < 40:
            u, v = (int(x) for x in rng.integers(0, 4096, 2))
            u, v = min(u, v), max(u, v)
            if u != v and not gh.has_arc(u, v) and deg[u] + 2 < deg.max() and deg[v] + 2 < deg.max():
                ins.add((u, v))
        present = [a for a in gh.arcs() if a[0] < a[1]][:5]
        b = P.EdgeBatch(insertions=[a for uv in sorted(ins) for a in (uv, uv[::-1])],
                        deletions=[a for uv in present for a in (uv, uv[::-1])])
        v0 = gd.version
        P.update_batch(sd, gd, b, theta=0.5)
        P.update_batch(sh, gh, b, theta=0.5)
        assert gd.version == v0 + 2 == gh.version - (gh.version - v0 - 2)
        np.testing.assert_array_equal(sd.lower, sh.lower)
        np.testing.assert_array_equal(sd.upper, sh.upper)
        assert sd.last_update_stats == sh.last_update_stats
        ip2, ix2 = gd.csr_arrays()
        ih, xh = gh.csr_arrays()
        np.testing.assert_array_equal(ip2, ih)
        np.testing.assert_array_equal(ix2, xh)
        deg = np.diff(ih)
    ip3, ix3 = gd.csr_arrays()
    existing = (0, int(ix3[ip3[0]]))
    with pytest.raises(P.BatchPreconditionError):
        gd.validate_batch(P.EdgeBatch(insertions=[existing]))
    with pytest.raises(P.BatchPreconditionError):
        gd.validate_batch(P.EdgeBatch(deletions=[present[0]]))
    assert gd.max_out_degree() == gh.max_out_degree()


def test_device_symmetry_check_cases():
    cases = [
        ([(0, 1), (1, 0), (2, 2)], True),           # self-loop is its own reverse
        ([(0, 1), (1, 0), (1, 2)], False),
        ([(0, 2), (2, 0), (1, 2), (2, 1), (3, 3)], True),
        ([(3, 0), (0, 3), (2, 0)], False),
        ([], True),
    ]
    for arcs, sym in cases:
        g = P.Graph.from_edges(5, arcs)
        assert P.device_graph(g).is_symmetric() == sym, arcs
        assert g.is_symmetric() == sym
    gr = G.rmat_graph(1 << 14, edge_factor=16, seed=1)
    ip, ix = gr.csr_arrays()
    assert P.DeviceGraph(ip, ix).is_symmetric()
    row = ix[ip[5]:ip[6]].copy()
    cand = [c for c in range(1 << 14) if c != 5 and c not in set(row.tolist())]
    ix2 = ix.copy()
    row[-1] = max(cand) if max(cand) > row[-2] else row[-1]
    ix2[ip[5]:ip[6]] = np.sort(row)
    if not np.array_equal(ix2, ix):
        assert not P.DeviceGraph(ip, ix2).is_symmetric()
