"""CUDA path vs the CPU oracle and the reference's golden vectors (B200).

Bar (north_star): identical certified order, iteration count and separated
fraction; bounds bit-identical where every row sum is sequential (rows no
longer than the split threshold -- all of them when the threshold is raised
above deg_max), else within 1e-12 relative.
"""
from __future__ import annotations

import hashlib

import numpy as np
import pytest

from oracle import katz_oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_1807_03847_b200")

RTOL = 1e-12   # north_star: "bounds within a 1e-12 relative tolerance"


def h16(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def to_graph(g0: O.CSRGraph) -> "P.Graph":
    return P.Graph.from_csr(g0.node_count, g0.indptr, g0.indices)


def crit(c):
    kind = c["kind"]
    if kind == "ranking":
        return P.Criterion.ranking(c["epsilon"])
    if kind == "topk":
        return P.Criterion.top_k(c["k"], c["epsilon"])
    if kind == "score":
        return P.Criterion.score(c["epsilon"])
    return P.Criterion.pair(c["u"], c["v"], c["epsilon"])


def assert_same_active(mine, ref, lower, key):
    mine, ref = np.sort(mine), np.sort(ref)
    if np.array_equal(mine, ref):
        return
    assert mine.size == ref.size, key
    np.testing.assert_array_equal(np.sort(lower[mine]), np.sort(lower[ref]), err_msg=key)


def test_small_golden_cases_bitwise(golden_index, small_cases):
    """Every small reference case: bitwise order/bounds/katz/levels/r."""
    for c in golden_index["small"]:
        key = c["key"]
        e = small_cases[f"{c['graph']}/edges"]
        g = P.Graph.from_edges(c["n"], e, undirected=False)
        st = P.init(g, crit(c), undirected=c["undirected"])
        assert st.alpha == c["alpha"] and st.gamma == c["gamma"], key
        res = P.run(st, g)
        assert res.iterations_used == c["r"], key
        np.testing.assert_array_equal(res.order, small_cases[key + "/order"], err_msg=key)
        np.testing.assert_array_equal(res.lower, small_cases[key + "/lower"], err_msg=key)
        np.testing.assert_array_equal(res.upper, small_cases[key + "/upper"], err_msg=key)
        np.testing.assert_array_equal(st.katz, small_cases[key + "/katz"], err_msg=key)
        np.testing.assert_array_equal(np.stack(list(st.levels)),
                                      small_cases[key + "/levels"], err_msg=key)
        assert_same_active(st.active, small_cases[key + "/active"], res.lower, key)
        assert res.separated_fraction == c["sepfrac"], key


@pytest.fixture(scope="module")
def c1():
    g0 = O.rmat_graph(65536, edge_factor=16, seed=42)
    return g0, to_graph(g0)


def test_C1_exact_digests_without_split(golden_index, c1):
    """Split threshold above deg_max: every row is one sequential sum, so the
    device reproduces the reference's digests bit for bit."""
    d = golden_index["digests"]["C1_topk100"]
    g0, g = c1
    dg = P.DeviceGraph(g0.indptr, g0.indices, split_threshold=1 << 20)
    g._device = (g.version, dg)
    st = P.init(g, P.Criterion.top_k(100, 1e-6), undirected=True)
    res = P.run(st, g)
    g._device = None
    assert res.iterations_used == d["r"]
    assert res.separated_fraction == d["sepfrac"]
    assert h16(res.order) == d["order"]
    assert h16(res.lower) == d["lower"] and h16(res.upper) == d["upper"]
    assert st.active.size == d["active"]


def test_C1_default_split_within_tolerance(golden_index, c1):
    d = golden_index["digests"]["C1_topk100"]
    g0, g = c1
    st = P.init(g, P.Criterion.top_k(100, 1e-6), undirected=True)
    info = st.device_graph.info()
    deg = np.diff(g0.indptr)
    assert info.heavy_rows == int((deg > info.split_threshold).sum()) >= 1
    assert info.max_out_degree == 9648
    res = P.run(st, g)
    ost = O.OracleState(g0, O.Crit("topk", 1e-6, k=100))
    ores = O.run(ost, g0)
    assert res.iterations_used == ores.iterations_used == d["r"]
    assert res.top(100) == d["top100"]
    np.testing.assert_array_equal(res.order, ores.order)
    np.testing.assert_allclose(res.lower, ores.lower, rtol=RTOL, atol=0)
    np.testing.assert_allclose(res.upper, ores.upper, rtol=RTOL, atol=0)
    assert res.separated_fraction == d["sepfrac"]
    assert sorted(st.active.tolist()) == sorted(ost.active.tolist())


def test_fixture_eps_sweep(golden_index):
    """Acceptance gate 08 on the ef8 fixture: r and separated fraction per eps."""
    d = golden_index["digests"]
    g0 = O.rmat_graph(65536, edge_factor=8, seed=42)
    g = to_graph(g0)
    for eps, r, frac in d["fixture_eps_sweep"]:
        st = P.init(g, P.Criterion.ranking(eps), undirected=True)
        res = P.run(st, g)
        assert (res.iterations_used, res.separated_fraction) == (r, frac), eps


def test_grid256_ranking_bitwise(golden_index):
    """Exact interior ties: order decided by rounding, so only bit-exact
    arithmetic reproduces it (SURVEY.md 8(c) parity fact 4)."""
    d = golden_index["digests"]["grid256_ranking1e-9"]
    g0 = O.grid_graph(256 * 256)
    g = to_graph(g0)
    st = P.init(g, P.Criterion.ranking(1e-9), undirected=True)
    res = P.run(st, g)
    assert res.iterations_used == d["r"] == 99
    assert h16(res.order) == d["order"]
    assert h16(res.lower) == d["lower"] and h16(res.upper) == d["upper"]
    assert res.separated_fraction == d["sepfrac"]


@pytest.mark.parametrize("split", [0, 64, 1 << 20])
def test_rmat_s12_topk_vs_oracle(golden_index, split):
    """Real Graph fixture of the golden set; segmentation thresholds vary."""
    d = golden_index["digests"]["rmat_s12_seed3_topk50"]
    g0 = O.rmat_graph(4096, edge_factor=16, seed=3)
    g = to_graph(g0)
    g._device = (g.version, P.DeviceGraph(g0.indptr, g0.indices, split_threshold=split))
    st = P.init(g, P.Criterion.top_k(50, 1e-9), undirected=True)
    res = P.run(st, g)
    assert res.iterations_used == d["r"]
    assert res.top(100) == d["top100"]
    assert res.separated_fraction == d["sepfrac"]
    if split == 1 << 20:
        assert h16(res.lower) == d["lower"] and h16(res.upper) == d["upper"]
        assert h16(res.order) == d["order"]
    else:
        ost = O.OracleState(g0, O.Crit("topk", 1e-9, k=50))
        ores = O.run(ost, g0)
        np.testing.assert_allclose(res.lower, ores.lower, rtol=RTOL, atol=0)
        np.testing.assert_allclose(res.upper, ores.upper, rtol=RTOL, atol=0)


def test_iterate_and_check_step_by_step():
    """iterate_once/check_converged individually agree with the oracle at
    every step, including the shrinking active set."""
    g0 = O.rmat_graph(8192, edge_factor=16, seed=11)
    g = to_graph(g0)
    st = P.init(g, P.Criterion.top_k(20, 1e-8), undirected=True)
    ost = O.OracleState(g0, O.Crit("topk", 1e-8, k=20))
    for _ in range(12):
        P.iterate_once(st, g)
        O.iterate_once(ost, g0)
        assert st.r == ost.r
        np.testing.assert_allclose(st.levels[-1], ost.levels[-1], rtol=RTOL, atol=0)
        np.testing.assert_allclose(st.katz, ost.katz, rtol=RTOL, atol=0)
        done = P.check_converged(st)
        odone = O.check_converged(ost)
        assert done == odone
        assert sorted(st.active.tolist()) == sorted(ost.active.tolist())
        # the sorted prefix is identical and in the same order
        k = min(20, st.active.size)
        assert st.active[:k].tolist() == ost.active[:k].tolist()
        if done:
            break
    assert done


def test_directed_graph_and_pair_score():
    rng = np.random.default_rng(4)
    n = 3000
    e = rng.integers(0, n, size=(20000, 2))
    g = P.Graph.from_edges(n, e[e[:, 0] != e[:, 1]])
    g0 = O.CSRGraph(n, *g.csr_arrays())
    for c, oc in [(P.Criterion.score(1e-9), O.Crit("score", 1e-9)),
                  (P.Criterion.pair(5, 17, 1e-7), O.Crit("pair", 1e-7, u=5, v=17)),
                  (P.Criterion.ranking(1e-5), O.Crit("ranking", 1e-5))]:
        st = P.init(g, c)
        res = P.run(st, g)
        ost = O.OracleState(g0, oc, undirected=False)
        ores = O.run(ost, g0)
        assert res.iterations_used == ores.iterations_used
        np.testing.assert_array_equal(res.lower, ores.lower)
        np.testing.assert_array_equal(res.upper, ores.upper)
        np.testing.assert_array_equal(res.order, ores.order)
        assert res.separated_fraction == ores.separated_fraction


def test_device_symmetry_check():
    g = P.Graph.from_edges(5, [(0, 1), (1, 2)], undirected=True)
    assert P.device_graph(g).is_symmetric()
    gd = P.Graph.from_edges(5, [(0, 1), (1, 2)])
    assert not P.device_graph(gd).is_symmetric()


def test_convergence_error_carries_iterations_and_gap():
    g = P.Graph.from_edges(6, [(i, j) for i in range(6) for j in range(i + 1, 6)],
                           undirected=True)
    st = P.init(g, P.Criterion.score(1e-10), undirected=True, max_iterations=2)
    with pytest.raises(P.ConvergenceError) as exc:
        P.run(st, g)
    assert exc.value.iterations == 2 and exc.value.gap > 1e-10


def test_stale_graph_rejected():
    g = P.Graph.from_edges(4, [(0, 1), (1, 2), (2, 3)], undirected=True)
    st = P.init(g, P.Criterion.ranking(1e-6))
    g.insert_arcs([(0, 2)])
    with pytest.raises(P.StateError):
        P.iterate_once(st, g)
    st2 = P.init(g, P.Criterion.ranking(1e-6))
    with pytest.raises(P.StateError):
        P.check_converged(st2)


def test_k_boundary_ties_are_detected_and_reported():
    """SURVEY.md 8(c) rule 4: on a cycle every node ties every other, so the
    top-2 cut drops tied nodes once their gap < eps -- where the reference's
    argpartition (engine.py:359) picks arbitrarily.  The state counts them
    and run() warns; the certified order is unaffected (node-id ties)."""
    n = 12
    g = P.Graph.from_edges(n, [(i, (i + 1) % n) for i in range(n)], undirected=True)
    st = P.init(g, P.Criterion.top_k(2, 1e-6), undirected=True)
    with pytest.warns(P.KBoundaryTieWarning):
        res = P.run(st, g)
    assert st.k_boundary_ties > 0
    assert list(res.order) == list(range(n))
    # R-MAT bounds never tie at the cut (SURVEY.md 8(c) margins)
    g0 = O.rmat_graph(4096, edge_factor=16, seed=3)
    g2 = P.Graph.from_csr(g0.node_count, g0.indptr, g0.indices)
    st2 = P.init(g2, P.Criterion.top_k(50, 1e-9), undirected=True)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("error", P.KBoundaryTieWarning)
        P.run(st2, g2)
    assert st2.k_boundary_ties == 0


@pytest.mark.parametrize("kind", ["topk", "ranking"])
def test_device_loop_cap_rerun_and_state(kind):
    """The device-driven run loops (TOPK batches of K1 + check, RANKING
    cached-pair chains) against the oracle's engine.run on the same graph:
    hitting max_iterations mid-batch raises ConvergenceError with the
    reference's iteration count and leaves exactly r + 1 levels; a second
    run on a converged state iterates once more and converges again, as
    engine.py:382-396 does; the state afterwards answers check_converged."""
    if kind == "topk":
        g0 = O.rmat_graph(1 << 14, edge_factor=16, seed=42)
        crit, ocrit = P.Criterion.top_k(100, 1e-6), O.Crit("topk", 1e-6, k=100)
    else:
        g0 = O.grid_graph(40 * 40)
        crit, ocrit = P.Criterion.ranking(1e-9), O.Crit("ranking", 1e-9)
    g = P.Graph.from_csr(g0.node_count, g0.indptr, g0.indices)
    ref = O.run(O.OracleState(g0, ocrit), g0)
    r = ref.iterations_used
    assert r > 3
    st = P.init(g, crit, undirected=True, max_iterations=r - 2)
    with pytest.raises(P.ConvergenceError) as ei:
        P.run(st, g)
    assert ei.value.iterations == r - 2 and st.r == r - 2 and len(st.levels) == r - 1
    st = P.init(g, crit, undirected=True)
    res = P.run(st, g)
    assert res.iterations_used == r and np.array_equal(res.order, ref.order)
    assert P.check_converged(st)
    res2 = P.run(st, g)
    assert res2.iterations_used == r + 1 and st.r == r + 1
    ost = O.OracleState(g0, ocrit)
    O.run(ost, g0)
    O.iterate_once(ost, g0)
    assert O.check_converged(ost)
    np.testing.assert_allclose(res2.lower, ost.lower, rtol=1e-12, atol=0)


@pytest.mark.parametrize("case,k", [("rmat12", 100), ("rmat14", 100), ("star", 100),
                                    ("rmat10", 600), ("rmat12", 1)])
def test_level1_check_shortcut_matches_the_general_check(case, k):
    """The TOPK check right after the first iteration of a fresh layout reads
    the winners, threshold and survivors off the degree order
    (k_topk_level1) and leaves the active set as the dense prefix [0, S)
    for the next check.  Against the general select (kb_tune chk.level1 0):
    the same r, active set (in order), bounds, order, separated fraction and
    boundary-tie count, bit for bit (the star's leaves all tie at the cut)."""
    from paper_1807_03847_b200 import _lib
    L = _lib.lib()
    if case.startswith("rmat"):
        n = 1 << int(case[4:])
        g0 = O.rmat_graph(n, edge_factor=8, seed=int(case[4:]))
        ip, ix = g0.indptr, g0.indices
    else:
        n = 300
        e = [(0, v) for v in range(1, n)]
        a = np.array(e + [(v, u) for u, v in e], dtype=np.int64)
        a = a[np.lexsort((a[:, 1], a[:, 0]))]
        ip = np.zeros(n + 1, dtype=np.int64)
        np.add.at(ip, a[:, 0] + 1, 1)
        ip = np.cumsum(ip)
        ix = a[:, 1].astype(np.int32)
    out = {}
    for flag in (0, 1):
        _lib.check(L.kb_tune(b"chk.level1", flag))
        try:
            g = P.Graph.from_csr(n, ip, ix)
            st = P.init(g, P.Criterion.top_k(k, 1e-6), undirected=True, max_iterations=500)
            res = P.run(st, g)
            out[flag] = (st.r, np.asarray(st.active).copy(), np.asarray(st.lower).copy(),
                         np.asarray(st.upper).copy(), np.asarray(res.order).copy(),
                         res.separated_fraction, st.k_boundary_ties)
        finally:
            _lib.check(L.kb_tune(b"chk.level1", 1))
    a0, a1 = out[0], out[1]
    assert a0[0] == a1[0]
    for x, y in zip(a0[1:5], a1[1:5]):
        np.testing.assert_array_equal(x, y)
    assert a0[5] == a1[5] and a0[6] == a1[6]


@pytest.mark.parametrize("bits", [40, 24, 8])
def test_prefix_result_sort_matches_the_full_sort(bits):
    """K3's prefix sort (a stable radix sort of the top varying key bits,
    then the out-of-order equal-prefix runs fixed; too many or too long runs
    fall back to the full sort) gives the full sort's order, sorted keys and
    separated-pair count bit for bit.  8 prefix bits force the fallback."""
    from paper_1807_03847_b200 import _lib
    L = _lib.lib()
    g0 = O.rmat_graph(1 << 18, edge_factor=8, seed=5)
    g = P.Graph.from_csr(g0.node_count, g0.indptr, g0.indices)
    out = {}
    for prefix in (0, 1):
        _lib.check(L.kb_tune(b"result.prefix_sort", prefix))
        _lib.check(L.kb_tune(b"result.prefix_bits", bits))
        _lib.check(L.kb_tune(b"result.prefix_exact_bits", 0))   # always prefix + fix-up
        try:
            st = P.init(g, P.Criterion.top_k(100, 1e-6), undirected=True)
            res = P.run(st, g)
            out[prefix] = (np.asarray(res.order).copy(), res.separated_fraction,
                           np.asarray(res.lower).copy())
        finally:
            _lib.check(L.kb_tune(b"result.prefix_sort", 1))
            _lib.check(L.kb_tune(b"result.prefix_bits", -1))     # back to the default
            _lib.check(L.kb_tune(b"result.prefix_exact_bits", 56))
    np.testing.assert_array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1]
    np.testing.assert_array_equal(out[0][2], out[1][2])
