"""Pin the CPU oracle against the reference's golden vectors (no GPU).

Fixtures were produced by running the reference package itself
(tests/golden/make_golden.py); the known-answer cases restate the
reference suite (pkg/tests/test_engine.py:79-138, :308-344).
"""
from __future__ import annotations

import hashlib

import numpy as np
import pytest

from oracle import katz_oracle as O


def h16(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def graph_from_edges(n, edges, undirected):
    # golden edges are the reference Graph.arcs(): already both directions
    return O.CSRGraph.from_edges(n, edges.reshape(-1, 2), undirected=False)


def assert_same_active(mine, ref, lower, key):
    """The reference's argpartition (engine.py:359) breaks exact ties at the
    k-th position arbitrarily; the oracle and the device break them by id.
    Sets must agree exactly, or -- when the cut falls inside a tie -- agree
    as multisets of lower bounds (same size, same values)."""
    mine, ref = np.sort(mine), np.sort(ref)
    if np.array_equal(mine, ref):
        return
    assert mine.size == ref.size, key
    np.testing.assert_array_equal(np.sort(lower[mine]), np.sort(lower[ref]), err_msg=key)


def crit_of(c):
    return O.Crit(c["kind"], c["epsilon"], k=c["k"], u=c["u"], v=c["v"])


def test_small_cases_bitwise(golden_index, small_cases):
    for c in golden_index["small"]:
        key = c["key"]
        g = graph_from_edges(c["n"], small_cases[f"{c['graph']}/edges"], c["undirected"])
        st = O.OracleState(g, crit_of(c), undirected=c["undirected"])
        assert st.alpha == c["alpha"] and st.gamma == c["gamma"], key
        assert st.max_iterations == c["max_iterations"], key
        res = O.run(st, g)
        assert res.iterations_used == c["r"], key
        np.testing.assert_array_equal(res.order, small_cases[key + "/order"], err_msg=key)
        np.testing.assert_array_equal(res.lower, small_cases[key + "/lower"], err_msg=key)
        np.testing.assert_array_equal(res.upper, small_cases[key + "/upper"], err_msg=key)
        np.testing.assert_array_equal(st.katz, small_cases[key + "/katz"], err_msg=key)
        np.testing.assert_array_equal(np.stack(st.levels), small_cases[key + "/levels"], err_msg=key)
        assert_same_active(st.active, small_cases[key + "/active"], res.lower, key)
        assert res.separated_fraction == c["sepfrac"], key


def test_pcg64_replica(golden_index):
    d = golden_index["digests"]
    s, inc = (int(x) for x in d["pcg64_seed42_state"])
    M = (1 << 64) - 1
    out = np.empty(64, dtype=np.uint64)
    O.lib().oracle_pcg64_raw(s >> 64, s & M, inc >> 64, inc & M, 0, 64, O._p(out))
    assert [int(x) for x in out] == d["pcg64_seed42_raw64"]
    # jump-ahead reproduces any window of the stream
    out2 = np.empty(10, dtype=np.uint64)
    O.lib().oracle_pcg64_raw(s >> 64, s & M, inc >> 64, inc & M, 37, 10, O._p(out2))
    assert [int(x) for x in out2] == d["pcg64_seed42_raw64"][37:47]


@pytest.mark.parametrize("ef", [8, 16])
def test_rmat_replica_matches_reference(golden_index, ef):
    d = golden_index["digests"]
    packed = O.rmat_packed(65536, edge_factor=ef, seed=42)
    assert packed.size == d[f"rmat_s16_ef{ef}_edges"]["count"]
    assert h16(packed) == d[f"rmat_s16_ef{ef}_edges"]["packed"]
    g = O.rmat_graph(65536, edge_factor=ef, seed=42)
    csr = d[f"rmat_s16_ef{ef}_csr"]
    assert g.nnz == csr["nnz"] and g.max_out_degree() == csr["dmax"]
    assert h16(g.indptr) == csr["indptr"] and h16(g.indices) == csr["indices"]
    assert g.is_symmetric()


def test_C1_digests(golden_index):
    d = golden_index["digests"]["C1_topk100"]
    g = O.rmat_graph(65536, edge_factor=16, seed=42)
    st = O.OracleState(g, O.Crit("topk", 1e-6, k=100))
    assert st.alpha == d["alpha"] and st.gamma == d["gamma"]
    res = O.run(st, g)
    assert res.iterations_used == d["r"] == 8
    assert res.separated_fraction == d["sepfrac"]
    assert h16(res.order.astype(np.int64)) == d["order"]
    assert h16(res.lower) == d["lower"] and h16(res.upper) == d["upper"]
    assert res.top(10) == d["top10"]
    assert st.active.size == d["active"]


def test_fixture_eps_sweep(golden_index):
    """Acceptance gate 08 (test_acceptance.py:368-383) on the ef8 fixture."""
    d = golden_index["digests"]
    g = O.rmat_graph(65536, edge_factor=8, seed=42)
    for eps, r, frac in d["fixture_eps_sweep"]:
        st = O.OracleState(g, O.Crit("ranking", eps))
        res = O.run(st, g)
        assert (res.iterations_used, res.separated_fraction) == (r, frac)
    fx = d["fixture_ranking1e-6"]
    st = O.OracleState(g, O.Crit("ranking", 1e-6))
    res = O.run(st, g)
    assert h16(res.order.astype(np.int64)) == fx["order"]
    assert h16(res.lower) == fx["lower"] and h16(res.upper) == fx["upper"]


def test_grid256_digests(golden_index):
    d = golden_index["digests"]["grid256_ranking1e-9"]
    g = O.grid_graph(256 * 256)
    st = O.OracleState(g, O.Crit("ranking", 1e-9))
    res = O.run(st, g)
    assert res.iterations_used == d["r"] == 99
    assert h16(res.order.astype(np.int64)) == d["order"]
    assert h16(res.lower) == d["lower"] and h16(res.upper) == d["upper"]


def test_matvec_threads_bitwise():
    """engine.py:184-187 / test_engine.py:356-365: thread count is invisible."""
    g = O.rmat_graph(4096, edge_factor=16, seed=3)
    x = np.random.default_rng(0).random(4096)
    y1 = O.csr_matvec(g, x, 1)
    for t in (2, 3, 8):
        np.testing.assert_array_equal(O.csr_matvec(g, x, t), y1)
    # strict sequential ascending order, the scipy csr_matvec semantics
    # (a plain loop: Python 3.12's sum() of floats is compensated)
    ref = np.zeros(4096)
    for i, (a, b) in enumerate(zip(g.indptr[:-1], g.indptr[1:])):
        acc = 0.0
        for v in x[g.indices[a:b]].tolist():
            acc += v
        ref[i] = acc
    np.testing.assert_array_equal(y1, ref)


def test_known_answers():
    # K3 at alpha=1/3 (test_engine.py:79-93)
    k3 = O.CSRGraph.from_edges(3, [(0, 1), (0, 2), (1, 2)], undirected=True)
    st = O.OracleState(k3, O.Crit("score", 1e-6), alpha=1 / 3)
    O.iterate_once(st, k3)
    assert np.all(st.levels[1] == 2 / 3) and np.all(st.katz == 2 / 3)
    np.testing.assert_allclose(st.lower, 8 / 9, rtol=1e-15)
    np.testing.assert_allclose(st.upper, 2.0, rtol=0, atol=5e-16)
    # K4 at alpha=.25 (:96-104)
    k4 = O.CSRGraph.from_edges(4, [(i, j) for i in range(4) for j in range(i + 1, 4)],
                               undirected=True)
    st = O.OracleState(k4, O.Crit("score", 1e-6), alpha=0.25)
    O.iterate_once(st, k4)
    assert np.all(st.upper == 3.0) and st.gap() == 2.0625
    # directed path at alpha=.5 terminates exactly (:120-128, :308-318)
    dp = O.CSRGraph.from_edges(3, [(0, 1), (1, 2)])
    st = O.OracleState(dp, O.Crit("score", 0.25), alpha=0.5, undirected=False)
    O.run(st, dp)
    np.testing.assert_array_equal(st.lower, [0.75, 0.5, 0.0])
    np.testing.assert_array_equal(st.upper, [0.75, 0.5, 0.0])
    assert not O.epsilon_separated(st, 1, 0) and O.epsilon_separated(st, 1, 2)


def test_separated_pairs_bruteforce():
    rng = np.random.default_rng(5)
    lower = rng.random(300).round(2)
    upper = lower + rng.random(300).round(2) * 0.1
    brute = int(sum((lower > u).sum() for u in upper))
    assert O.separated_pairs(lower, upper) == brute


def test_dynamic_oracle_matches_reference(golden_index, dynamic_cases):
    for c in golden_index["dynamic"]:
        name = c["name"]
        edges = dynamic_cases[f"{name}/edges0"]
        g = O.AdjGraph(c["n"], [tuple(e) for e in edges.tolist()])
        crit = O.Crit(c["kind"], c["epsilon"], k=c["k"])
        st = O.OracleState(g, crit, alpha=c["alpha"], undirected=c["undirected"])
        O.run(st, g)
        for i, step in enumerate(c["steps"]):
            p = f"{name}/b{i}"
            stats = O.update_batch(st, g, dynamic_cases[p + "/ins"].tolist(),
                                   dynamic_cases[p + "/del"].tolist(), theta=c["theta"])
            assert st.r == step["r"], p
            np.testing.assert_array_equal(st.katz, dynamic_cases[p + "/katz"], err_msg=p)
            np.testing.assert_array_equal(st.lower, dynamic_cases[p + "/lower"], err_msg=p)
            np.testing.assert_array_equal(st.upper, dynamic_cases[p + "/upper"], err_msg=p)
            assert stats.level_sizes == step["level_sizes"], p
            assert stats.visited == step["visited"] and stats.seeds == step["seeds"], p
            assert stats.aborted_level == step["aborted_level"], p
            assert stats.reactivated == step["reactivated"], p
            assert_same_active(st.active, dynamic_cases[p + "/active"], st.lower, p)


def test_lowmem_rmat_generator_equals_pinned_generator():
    """The scale-27 golden build (tests/golden/make_c3_golden.py) uses the
    low-memory sampler: it must yield the same CSR as the pinned one."""
    a = O.rmat_graph(1 << 14, edge_factor=16, seed=42)
    for t in (1, 3, 8):
        b = O.rmat_graph_lowmem(1 << 14, edge_factor=16, seed=42, threads=t)
        assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
