"""CPU-only checks of the boundary and the host-side logic (no GPU needed)."""
from __future__ import annotations

import ctypes
import math
import os
import re

import numpy as np
import pytest

import paper_1807_03847_b200 as P
from paper_1807_03847_b200 import _lib
from oracle import katz_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "katzb200.h")).read()
    return sorted(set(re.findall(r"\b(kb_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    for name in syms:
        assert hasattr(L, name), name
    # the ctypes table covers the header exactly
    assert sorted(_lib.SIGNATURES) == syms


def test_library_reports_errors_without_gpu():
    L = _lib.lib()
    assert L.kb_version() >= 10000
    h = ctypes.c_void_p()
    rc = L.kb_graph_create(0, 3, 1, None, None, 0, -1, ctypes.byref(h))
    assert rc == _lib.KB_EPARAM and "NULL" in _lib.last_error()
    with pytest.raises(P.ParameterError):
        _lib.check(rc)


def test_parameter_plumbing_matches_reference_expressions():
    # engine.py:96-119, :286-293 restated; compare with the oracle's copy
    for d in (0, 1, 3, 9648, 406877):
        g = P.Graph.from_edges(d + 2, [(0, i) for i in range(1, d + 1)], undirected=True)
        assert P.default_alpha(g) == O.default_alpha(d)
        a = P.default_alpha(g)
        assert P.tail_gamma(a, d) == O.tail_gamma(a, d)
        for eps in (1e-1, 1e-6, 1e-12):
            assert P.default_iteration_cap(a, d, eps) == O.iteration_cap(a, d, eps)
    # C1 values from SURVEY.md 8(a) a2
    a = 1.0 / (1.0 + 9648)
    assert a == 0.00010363768266141569
    assert P.tail_gamma(a, 9648) == 93093551.99999869
    assert P.default_iteration_cap(a, 9648, 1e-6) == 1332990


@pytest.mark.parametrize("alpha", [0.0, -0.1, 0.25, 0.3, float("nan"), float("inf")])
def test_validate_alpha_rejects(alpha):
    with pytest.raises(P.ParameterError):
        P.validate_alpha(alpha, 4)


def test_validate_alpha_accepts_open_interval():
    P.validate_alpha(0.2499999, 4)
    P.validate_alpha(1e-9, 4)
    P.validate_alpha(0.999, 0)
    with pytest.raises(P.ParameterError):
        P.validate_alpha(1.0, 0)


def test_criterion_validation():
    with pytest.raises(P.ParameterError):
        P.Criterion.ranking(0.0)
    with pytest.raises(P.ParameterError):
        P.Criterion.top_k(0, 1e-6)
    with pytest.raises(P.ParameterError):
        P.Criterion.pair(2, 2, 1e-6)
    with pytest.raises(P.ParameterError):
        P.Criterion("nonsense")
    c = P.Criterion.top_k(5)
    assert (c.kind, c.k, c.epsilon) == ("topk", 5, 1e-6)


def test_init_rejects_bad_shapes_before_touching_the_device():
    g = P.Graph.from_edges(4, [(0, 1), (1, 2), (2, 3)], undirected=True)
    with pytest.raises(P.ParameterError):
        P.init(g, P.Criterion.top_k(5, 1e-6))
    with pytest.raises(P.ParameterError):
        P.init(g, P.Criterion.pair(0, 7))
    with pytest.raises(P.ParameterError):
        P.init(g, P.Criterion.ranking(1e-6), threads=0)
    gd = P.Graph.from_edges(3, [(0, 1)])
    with pytest.raises(P.ParameterError):
        P.init(gd, P.Criterion.ranking(1e-6), undirected=True)
    with pytest.raises(P.ParameterError):
        P.init(P.Graph(0), P.Criterion.ranking(1e-6))


def test_graph_store_matches_oracle_csr():
    g0 = O.rmat_graph(4096, edge_factor=16, seed=3)
    rows = np.repeat(np.arange(4096), np.diff(g0.indptr))
    e = np.stack([rows, g0.indices], 1)
    g = P.Graph.from_edges(4096, e[rows < g0.indices], undirected=True)
    ip, ix = g.csr_arrays()
    np.testing.assert_array_equal(ip, g0.indptr)
    np.testing.assert_array_equal(ix, g0.indices)
    assert g.is_symmetric() and g.max_out_degree() == g0.max_out_degree()
    v = int(np.argmax(np.diff(ip)))
    assert sorted(g.in_neighbors(v)) == sorted(g.out_neighbors(v))


def test_graph_mutation_and_batch_rules():
    g = P.Graph.from_edges(6, [(i, (i + 1) % 6) for i in range(6)], undirected=True)
    v0 = g.version
    with pytest.raises(P.BatchPreconditionError):
        g.validate_batch(P.EdgeBatch(insertions=[(0, 1)]))
    with pytest.raises(P.BatchPreconditionError):
        g.validate_batch(P.EdgeBatch(deletions=[(0, 3)]))
    with pytest.raises(P.BatchPreconditionError):
        P.EdgeBatch(insertions=[(0, 3), (0, 3)]).validate_shape()
    with pytest.raises(P.BatchPreconditionError):
        P.EdgeBatch(insertions=[(0, 3)], deletions=[(0, 3)]).validate_shape()
    with pytest.raises(P.NodeRangeError):
        g.validate_batch(P.EdgeBatch(insertions=[(0, 9)]))
    assert P.EdgeBatch(insertions=[(0, 3), (3, 0)]).is_symmetric()
    assert not P.EdgeBatch(insertions=[(0, 3)]).is_symmetric()
    g.apply_batch(P.EdgeBatch(insertions=[(0, 3), (3, 0)], deletions=[(0, 1), (1, 0)]))
    assert g.version == v0 + 2
    assert g.has_arc(0, 3) and not g.has_arc(0, 1)
    assert sorted(g.out_neighbors(0)) == [3, 5]
    assert g.arc_count == 12


def test_generator_pcg_state_and_thresholds():
    from paper_1807_03847_b200 import generators as G
    st = G.pcg64_state(42)
    ref = np.random.default_rng(42).bit_generator.state["state"]
    assert (int(st[0]) << 64 | int(st[1])) == int(ref["state"])
    assert (int(st[2]) << 64 | int(st[3])) == int(ref["inc"])
