"""The reference suite's engine and acceptance behaviours, restated against
the device engine (pkg/tests/test_engine.py, test_acceptance.py).

Exact scores come from a dense solve, (I - alpha*A) z = 1, katz = z - 1,
as the reference's dense_oracle does (baselines.py:132-154).
"""
from __future__ import annotations

import math
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_1807_03847_b200")


# ---- graph builders (same families as pkg/tests/builders.py)

def complete(n):
    return P.Graph.from_edges(n, [(i, j) for i in range(n) for j in range(i + 1, n)],
                              undirected=True)


def star(n):
    return P.Graph.from_edges(n, [(0, i) for i in range(1, n)], undirected=True)


def path(n):
    return P.Graph.from_edges(n, [(i, i + 1) for i in range(n - 1)], undirected=True)


def cycle(n):
    return P.Graph.from_edges(n, [(i, (i + 1) % n) for i in range(n)], undirected=True)


def grid(rows, cols):
    e = []
    for r in range(rows):
        for c in range(cols):
            v = r * cols + c
            if c + 1 < cols:
                e.append((v, v + 1))
            if r + 1 < rows:
                e.append((v, v + cols))
    return P.Graph.from_edges(rows * cols, e, undirected=True)


def er(n, p, seed, undirected=True):
    rng = random.Random(seed)
    e = []
    for i in range(n):
        for j in range(i + 1 if undirected else 0, n):
            if i != j and rng.random() < p:
                e.append((i, j))
    return P.Graph.from_edges(n, e, undirected=undirected)


def exact_katz(g, alpha):
    n = g.node_count
    A = np.zeros((n, n))
    ip, ix = g.csr_arrays()
    for v in range(n):
        A[v, ix[ip[v]:ip[v + 1]]] = 1.0
    z = np.linalg.solve(np.eye(n) - alpha * A, np.ones(n))
    return z - 1.0


# ---- frozen values (test_engine.py:79-138)

def test_triangle_first_level_exact():
    g = complete(3)
    st = P.init(g, P.Criterion.score(1e-6), alpha=1 / 3, undirected=True)
    P.iterate_once(st, g)
    assert st.r == 1
    np.testing.assert_array_equal(st.levels[1], 2 / 3)
    np.testing.assert_array_equal(st.katz, 2 / 3)
    np.testing.assert_allclose(st.lower, 8 / 9, rtol=1e-15)
    np.testing.assert_allclose(st.upper, 2.0, rtol=0, atol=5e-16)


def test_k4_upper_is_exact_katz():
    g = complete(4)
    st = P.init(g, P.Criterion.score(1e-6), alpha=0.25, undirected=True)
    P.iterate_once(st, g)
    np.testing.assert_array_equal(st.upper, 3.0)
    assert st.gap() == 2.0625


def test_star_converged_values():
    g = star(4)
    st = P.init(g, P.Criterion.score(1e-12), alpha=0.25, undirected=True)
    P.run(st, g)
    ex = np.array([15 / 13, 7 / 13, 7 / 13, 7 / 13])
    np.testing.assert_allclose(st.katz, ex, rtol=1e-11)
    assert np.all(st.lower <= ex + 1e-15) and np.all(st.upper >= ex - 1e-15)


def test_directed_path_terminates_exactly():
    g = P.Graph.from_edges(3, [(0, 1), (1, 2)])
    st = P.init(g, P.Criterion.score(1e-9), alpha=0.5)
    P.run(st, g)
    np.testing.assert_allclose(st.katz, [0.75, 0.5, 0.0], rtol=0, atol=1e-15)
    np.testing.assert_array_equal(st.lower, st.katz)


def test_edgeless_graph_all_zero():
    g = P.Graph.from_edges(4, [])
    res = P.run(P.init(g, P.Criterion.ranking(1e-6)), g)
    assert res.iterations_used == 1
    np.testing.assert_array_equal(res.upper, 0.0)
    assert list(res.order) == [0, 1, 2, 3]


# ---- invariants (test_engine.py:143-191, test_acceptance.py gates 01-03)

def test_bounds_bracket_dense_solution():
    viol = 0
    for seed in range(8):
        g = er(30, 0.15, seed=seed)
        alpha = P.default_alpha(g)
        exact = exact_katz(g, alpha)
        st = P.init(g, P.Criterion.score(1e-9), alpha=alpha, undirected=True)
        slack = 1e-12 * (1.0 + np.abs(exact))
        for _ in range(12):
            P.iterate_once(st, g)
            viol += int(np.sum(st.lower > exact + slack)) + int(np.sum(st.upper < exact - slack))
    assert viol == 0


def test_complete_graph_upper_bound_sharp():
    worst = 0.0
    for n in range(3, 21):
        for delta in (0.5, 0.8):
            alpha = delta / (n - 1)
            exact = delta / (1.0 - delta)
            g = complete(n)
            st = P.init(g, P.Criterion.score(1e-9), alpha=alpha, undirected=True)
            for _ in range(6):
                P.iterate_once(st, g)
                worst = max(worst, float(np.max(np.abs(st.upper - exact))) / exact)
    assert worst < 1e-12


def test_bounds_monotone():
    g = grid(6, 6)
    st = P.init(g, P.Criterion.score(1e-9), undirected=True)
    pl, pu = st.lower.copy(), st.upper.copy()
    for _ in range(15):
        P.iterate_once(st, g)
        assert np.all(st.lower >= pl - 1e-15) and np.all(st.upper <= pu + 1e-15)
        pl, pu = st.lower.copy(), st.upper.copy()


def test_undirected_lower_adds_tail_step():
    g = cycle(6)
    st = P.init(g, P.Criterion.score(1e-9), undirected=True)
    P.iterate_once(st, g)
    np.testing.assert_array_equal(st.lower, st.katz + st.alpha * st.levels[1])


# ---- criteria (test_engine.py:196-318)

def test_pair_criterion_stops_early_and_orients():
    g = star(30)
    sp = P.init(g, P.Criterion.pair(0, 7, 1e-6), undirected=True)
    P.run(sp, g)
    sf = P.init(g, P.Criterion.ranking(1e-6), undirected=True)
    P.run(sf, g)
    assert sp.r <= sf.r and P.epsilon_separated(sp, 0, 7)
    g6 = star(6)
    s3 = P.init(g6, P.Criterion.pair(3, 0, 1e-6), undirected=True)
    P.run(s3, g6)
    assert s3.lower[0] > s3.upper[3] - 1e-6


def test_topk_shrinks_and_agrees_with_ranking():
    g = er(60, 0.1, seed=21)
    st = P.init(g, P.Criterion.top_k(5, 1e-8), undirected=True)
    prev = st.active.size
    for _ in range(st.max_iterations):
        P.iterate_once(st, g)
        done = P.check_converged(st)
        assert st.active.size <= prev
        prev = st.active.size
        if done:
            break
    g2 = er(50, 0.12, seed=4)
    rk = P.run(P.init(g2, P.Criterion.top_k(8, 1e-9), undirected=True), g2)
    rr = P.run(P.init(g2, P.Criterion.ranking(1e-9), undirected=True), g2)
    exact = exact_katz(g2, P.default_alpha(g2))
    order = np.lexsort((np.arange(50), -exact))
    for a, b in zip(rk.top(8), order[:8]):
        assert a == b or abs(exact[a] - exact[b]) < 1e-9
    for a, b in zip(rr.order, order):
        assert a == b or abs(exact[a] - exact[b]) < 1e-9


def test_result_frozen_sorted_and_ties_by_id():
    res = P.run(P.init(star(7), P.Criterion.ranking(1e-6), undirected=True), star(7))
    assert res.order[0] == 0 and np.all(np.diff(res.lower[res.order]) <= 0)
    with pytest.raises(ValueError):
        res.lower[0] = 99.0
    g = cycle(5)
    assert list(P.run(P.init(g, P.Criterion.ranking(1e-6), undirected=True), g).order) == \
        [0, 1, 2, 3, 4]


def test_iteration_cap_formula_and_error():
    g = complete(4)
    lo = P.init(g, P.Criterion.score(1e-2), undirected=True)
    hi = P.init(g, P.Criterion.score(1e-12), undirected=True)
    assert hi.max_iterations > lo.max_iterations
    rho = lo.alpha * 3
    assert lo.max_iterations == max(1, 10 * math.ceil(math.log(1e2) / math.log(1 / rho)))
    g6 = complete(6)
    st = P.init(g6, P.Criterion.score(1e-10), undirected=True, max_iterations=2)
    with pytest.raises(P.ConvergenceError) as e:
        P.run(st, g6)
    assert e.value.iterations == 2 and e.value.gap > 1e-10


def test_epsilon_separation_strict_and_symmetric_ties():
    g = star(4)
    st = P.init(g, P.Criterion.ranking(1e-6), undirected=True)
    P.run(st, g)
    assert P.epsilon_separated(st, 0, 1) and P.epsilon_separated(st, 1, 2)
    assert P.epsilon_separated(st, 2, 1) and not P.epsilon_separated(st, 1, 0)
    d = P.Graph.from_edges(3, [(0, 1), (1, 2)])
    s2 = P.init(d, P.Criterion.score(0.25), alpha=0.5)
    P.run(s2, d)
    np.testing.assert_array_equal(s2.upper, [0.75, 0.5, 0.0])
    assert not P.epsilon_separated(s2, 1, 0) and P.epsilon_separated(s2, 1, 2)
    with pytest.raises(P.ParameterError):
        P.epsilon_separated(s2, 0, 9)


def test_separated_fraction_exact_counts():
    st = P.init(star(4), P.Criterion.ranking(1e-4), undirected=True)
    P.run(st, star(4))
    assert P.separated_fraction(st) == 0.5
    for seed in range(6):
        g = er(25, 0.15, seed=seed)
        s = P.init(g, P.Criterion.score(1e-5), undirected=True)
        P.run(s, g)
        n = g.node_count
        brute = sum(1 for v in range(n) for w in range(n)
                    if v != w and s.lower[w] > s.upper[v])
        assert P.separated_fraction(s) == brute / (n * (n - 1) // 2)
    one = P.Graph.from_edges(1, [])
    s1 = P.init(one, P.Criterion.ranking(1e-6))
    P.run(s1, one)
    assert P.separated_fraction(s1) == 1.0


def test_threads_argument_is_invisible():
    g = er(120, 0.06, seed=17)
    r1 = P.run(P.init(g, P.Criterion.ranking(1e-8), undirected=True, threads=1), g)
    r8 = P.run(P.init(g, P.Criterion.ranking(1e-8), undirected=True, threads=8), g)
    assert r1.iterations_used == r8.iterations_used
    np.testing.assert_array_equal(r1.lower, r8.lower)
    np.testing.assert_array_equal(r1.order, r8.order)


def test_reference_graph_type_is_accepted():
    """A duck-typed graph (the reference's Graph surface) goes through the
    device path unchanged (engine.py:98,189,257,263,270,302)."""
    class Duck:
        def __init__(self, g):
            self._g = g
            self.node_count = g.node_count
            self.version = 7

        def max_out_degree(self):
            return self._g.max_out_degree()

        def is_symmetric(self):
            return self._g.is_symmetric()

        def out_csr(self):
            return self._g.out_csr()

    g = er(40, 0.1, seed=3)
    d = Duck(g)
    a = P.run(P.init(d, P.Criterion.top_k(5, 1e-9), undirected=True), d)
    b = P.run(P.init(g, P.Criterion.top_k(5, 1e-9), undirected=True), g)
    np.testing.assert_array_equal(a.order, b.order)
    np.testing.assert_array_equal(a.upper, b.upper)
