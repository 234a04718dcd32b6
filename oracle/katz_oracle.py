"""CPU oracle for the bounded-Katz hot path -- TEST INFRASTRUCTURE ONLY.

This module restates, in numpy plus the plain-C matvec of ``oracle.c``, the
reference algorithm of ``katzbounds`` (/root/reference/pkg/src/katzbounds).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs
(``cpu_baseline`` and ``--impl reference``) may import it, and only as the
checker or as the timed CPU baseline.  The product package
``paper_1807_03847_b200`` never imports it and has no CPU fallback.

Parity pinning: the oracle is checked (tests/test_oracle.py) against

* golden vectors produced by running the reference itself in the build
  container (tests/golden/, script tests/golden/make_golden.py);
* the known-answer tests of the reference suite (test_engine.py:79-138,
  :308-318, :323-344) restated in tests/test_oracle.py;
* the sha256 digests SURVEY.md section 8(c) records for C1 and the
  s16/ef8 acceptance fixture.

Every function cites the reference lines it restates.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


def build() -> str:
    """Compile oracle.c into oracle/_build/liboracle.so (make)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        i64, u64, dp = ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p
        L.oracle_csr_matvec.argtypes = [i64, dp, dp, dp, dp, ctypes.c_int]
        L.oracle_csr_matvec.restype = ctypes.c_int
        L.oracle_pcg64_raw.argtypes = [u64, u64, u64, u64, u64, i64, dp]
        L.oracle_pcg64_raw.restype = None
        L.oracle_rmat_pairs.argtypes = [u64, u64, u64, u64, ctypes.c_int, i64,
                                        ctypes.c_double, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_int, dp, dp, dp]
        L.oracle_rmat_pairs.restype = i64
        L.oracle_csr_from_packed.argtypes = [i64, i64, dp, dp, dp]
        L.oracle_csr_from_packed.restype = ctypes.c_int
        L.oracle_rmat_packed_lowmem.argtypes = [u64, u64, u64, u64, ctypes.c_int,
                                                i64, ctypes.c_double,
                                                ctypes.c_double, ctypes.c_double,
                                                ctypes.c_int, dp]
        L.oracle_rmat_packed_lowmem.restype = i64
        L.oracle_unique_sorted_inplace.argtypes = [i64, dp]
        L.oracle_unique_sorted_inplace.restype = i64
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------- CSR graph

class CSRGraph:
    """Duck-typed static graph the reference engine accepts.

    Surface used by engine.py: node_count, version, max_out_degree(),
    is_symmetric(), out_csr() (engine.py:98,189,257,263,270,302).  The CSR
    is the canonical sorted-row 0/1 snapshot of graph.py:177-197.
    """

    def __init__(self, n: int, indptr: np.ndarray, indices: np.ndarray,
                 symmetric: bool | None = None):
        self.node_count = int(n)
        self.indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        self.indices = np.ascontiguousarray(indices, dtype=np.int32)
        self.version = 1
        self._sym = symmetric
        self._csr = None

    @property
    def nnz(self) -> int:
        return int(self.indptr[-1])

    def out_degrees(self) -> np.ndarray:
        return np.diff(self.indptr)

    def max_out_degree(self) -> int:
        return int(self.out_degrees().max()) if self.node_count else 0

    def is_symmetric(self) -> bool:
        if self._sym is None:
            n = self.node_count
            rows = np.repeat(np.arange(n, dtype=np.int64), self.out_degrees())
            fwd = np.sort(rows * n + self.indices)
            bwd = np.sort(self.indices.astype(np.int64) * n + rows)
            self._sym = bool(np.array_equal(fwd, bwd))
        return self._sym

    def out_csr(self):
        """scipy view for running the *reference* engine on this graph."""
        if self._csr is None:
            from scipy import sparse
            data = np.ones(self.nnz, dtype=np.float64)
            self._csr = sparse.csr_matrix((data, self.indices, self.indptr),
                                          shape=(self.node_count,) * 2)
        return self._csr

    @classmethod
    def from_edges(cls, n: int, edges, undirected: bool = False) -> "CSRGraph":
        """Graph.from_edges (graph.py:101-116): duplicate arcs collapse."""
        e = np.asarray(list(edges) if not isinstance(edges, np.ndarray) else edges,
                       dtype=np.int64).reshape(-1, 2)
        src, dst = e[:, 0], e[:, 1]
        if undirected:
            src, dst = np.concatenate([src, dst]), np.concatenate([dst, src])
        key = np.unique(src * n + dst)
        rows, cols = key // n, key % n
        indptr = np.zeros(n + 1, dtype=np.int64)
        np.add.at(indptr, rows + 1, 1)
        np.cumsum(indptr, out=indptr)
        return cls(n, indptr, cols.astype(np.int32))


def csr_matvec(g: CSRGraph, x: np.ndarray, threads: int = 1) -> np.ndarray:
    """KatzState._matvec (engine.py:181-208) via oracle.c's sequential sum."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(g.node_count, dtype=np.float64)
    lib().oracle_csr_matvec(g.node_count, _p(g.indptr), _p(g.indices), _p(x),
                            _p(y), int(threads))
    return y


# ---------------------------------------------------------------- generators

def rmat_packed(n: int, edge_factor: int = 8, seed: int = 0,
                quadrants=(0.57, 0.19, 0.19, 0.05), threads: int | None = None
                ) -> np.ndarray:
    """generate.rmat_edges (generate.py:55-81) as sorted unique lo*n+hi keys.

    The draw stream is numpy's PCG64 from default_rng(seed); oracle.c
    replays it with jump-ahead so the sampling runs on all host threads.
    """
    if not (n >= 2 and (n & (n - 1)) == 0):
        raise ValueError("rmat needs a power-of-two node count >= 2")
    a, b, c, _ = quadrants
    ab = a + b            # same Python float expressions as generate.py:73-74
    abc = a + b + c
    scale = n.bit_length() - 1
    m = n * edge_factor
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    M = (1 << 64) - 1
    src = np.empty(m, dtype=np.int64)
    dst = np.empty(m, dtype=np.int64)
    packed = np.empty(m, dtype=np.int64)
    t = threads or os.cpu_count() or 1
    w = lib().oracle_rmat_pairs(s >> 64, s & M, inc >> 64, inc & M, scale, m,
                                a, ab, abc, t, _p(src), _p(dst), _p(packed))
    del src, dst
    return _sorted_unique(packed[:w])


def _sorted_unique(a: np.ndarray) -> np.ndarray:
    """np.unique (generate.py:80) as sort + mask: identical result; numpy
    2.3's np.unique is pathologically slow on large int64 arrays here."""
    a = np.sort(a)
    if a.size:
        keep = np.empty(a.size, dtype=bool)
        keep[0] = True
        np.not_equal(a[1:], a[:-1], out=keep[1:])
        a = a[keep]
    return a


def rmat_graph(n: int, edge_factor: int = 8, seed: int = 0) -> CSRGraph:
    """Graph.from_edges(n, generate('rmat', ...), undirected=True)."""
    packed = rmat_packed(n, edge_factor=edge_factor, seed=seed)
    indptr = np.empty(n + 1, dtype=np.int64)
    indices = np.empty(2 * packed.size, dtype=np.int32)
    lib().oracle_csr_from_packed(n, packed.size, _p(packed), _p(indptr),
                                 _p(indices))
    return CSRGraph(n, indptr, indices, symmetric=True)


def rmat_graph_lowmem(n: int, edge_factor: int = 8, seed: int = 0,
                      threads: int | None = None) -> CSRGraph:
    """rmat_graph with peak host memory ~ 8*m + 4*nnz bytes (scale 27 on a
    64 GB host): the sampler writes packed keys directly (no src/dst
    scratch), then an in-place sort + unique.  Same unique key set, hence
    the same CSR, as rmat_graph / generate.py:55-81."""
    if not (n >= 2 and (n & (n - 1)) == 0):
        raise ValueError("rmat needs a power-of-two node count >= 2")
    a, b, c, _ = (0.57, 0.19, 0.19, 0.05)
    ab = a + b
    abc = a + b + c
    scale = n.bit_length() - 1
    m = n * edge_factor
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    M = (1 << 64) - 1
    packed = np.empty(m, dtype=np.int64)
    t = threads or os.cpu_count() or 1
    w = lib().oracle_rmat_packed_lowmem(s >> 64, s & M, inc >> 64, inc & M,
                                        scale, m, a, ab, abc, t, _p(packed))
    view = packed[:w]
    view.sort()
    w = lib().oracle_unique_sorted_inplace(w, _p(view))
    indptr = np.empty(n + 1, dtype=np.int64)
    indices = np.empty(2 * w, dtype=np.int32)
    lib().oracle_csr_from_packed(n, w, _p(packed), _p(indptr), _p(indices))
    del packed, view
    return CSRGraph(n, indptr, indices, symmetric=True)


def grid_graph(n: int) -> CSRGraph:
    """generate.grid_edges (generate.py:38-52), loaded undirected."""
    cols = max(1, math.isqrt(n))
    i = np.arange(n, dtype=np.int64)
    right = ((i + 1) % cols != 0) & (i + 1 < n)
    down = i + cols < n
    e = np.concatenate([np.stack([i[right], i[right] + 1], 1),
                        np.stack([i[down], i[down] + cols], 1)])
    g = CSRGraph.from_edges(n, e, undirected=True)
    g._sym = True
    return g


# ---------------------------------------------------------------- engine

RANKING, TOPK, SCORE, PAIR = "ranking", "topk", "score", "pair"


@dataclass(frozen=True)
class Crit:
    """Criterion (engine.py:36-83) without the validation."""
    kind: str
    epsilon: float = 1e-6
    k: int | None = None
    u: int | None = None
    v: int | None = None


def default_alpha(d: int) -> float:
    """engine.py:96-99."""
    return 1.0 / (1.0 + d) if d > 0 else 0.5


def tail_gamma(alpha: float, d: int) -> float:
    """engine.py:116-119."""
    return d / (1.0 - alpha * d) if d > 0 else 0.0


def iteration_cap(alpha: float, d: int, eps: float) -> int:
    """engine.py:286-293."""
    rho = alpha * d
    if rho <= 0.0:
        return 64
    return max(1, 10 * math.ceil(math.log(1.0 / eps) / math.log(1.0 / rho)))


class OracleState:
    """KatzState (engine.py:124-177)."""

    def __init__(self, g: CSRGraph, crit: Crit, alpha: float | None = None,
                 undirected: bool = True, threads: int = 1,
                 keep_all_levels: bool = True, max_iterations: int | None = None):
        n = g.node_count
        d = g.max_out_degree()
        self.alpha = float(default_alpha(d) if alpha is None else alpha)
        self.gamma = tail_gamma(self.alpha, d)
        self.n = n
        self.crit = crit
        self.epsilon = crit.epsilon
        self.undirected = undirected
        self.threads = threads
        self.keep_all_levels = keep_all_levels
        self.max_iterations = (iteration_cap(self.alpha, d, crit.epsilon)
                               if max_iterations is None else max_iterations)
        self.r = 0
        self.levels = [np.ones(n)]                     # engine.py:147
        self.katz = np.zeros(n)                        # :148
        self.lower = np.zeros(n)                       # :149
        self.upper = np.full(n, self.alpha * self.gamma)  # :151
        self.active = np.arange(n, dtype=np.int64)     # :152
        self.last_update_stats = None

    def gap(self) -> float:
        return float(np.max(self.upper - self.lower)) if self.n else 0.0


def iterate_once(st: OracleState, g: CSRGraph) -> None:
    """engine.py:296-319 (numpy elementwise order: no FMA anywhere)."""
    alpha = st.alpha
    w_new = alpha * csr_matvec(g, st.levels[-1], st.threads)
    st.r += 1
    st.katz += w_new
    tail = alpha * w_new
    st.lower = st.katz + tail if st.undirected else st.katz.copy()
    st.upper = st.katz + tail * st.gamma
    st.levels.append(w_new)
    if not st.keep_all_levels and len(st.levels) > 2:
        del st.levels[0]


def epsilon_separated(st: OracleState, w: int, v: int) -> bool:
    """engine.py:322-330."""
    return bool(st.lower[w] > st.upper[v] - st.epsilon)


def check_converged(st: OracleState) -> bool:
    """engine.py:333-379.

    argpartition picks arbitrarily among exact ties at position k-1
    (engine.py:359); the oracle instead takes the top k by (-lower, id),
    which is what the device path does.  The threshold value, the sorted
    prefix and the survivor *set* are identical whenever the tie does not
    straddle the cut with gap < eps (SURVEY.md 8(c) rule 4); only the order
    of the survivors inside `active` may differ, and it is not observable.
    """
    kind = st.crit.kind
    eps = st.epsilon
    if kind == SCORE:
        return bool(np.max(st.upper - st.lower) < eps)
    if kind == PAIR:
        u, v = st.crit.u, st.crit.v
        if (st.lower[u], -u) >= (st.lower[v], -v):
            w, x = u, v
        else:
            w, x = v, u
        return epsilon_separated(st, w, x)
    k = st.n if kind == RANKING else st.crit.k
    m = st.active
    if m.size > k:
        order = np.lexsort((m, -st.lower[m]))
        top_ids = m[order[:k]]
        rest = np.sort(m[order[k:]])
    else:
        top_ids = m
        rest = np.empty(0, dtype=np.int64)
    prefix = top_ids[np.lexsort((top_ids, -st.lower[top_ids]))]
    threshold = st.lower[prefix[-1]]
    if rest.size:
        surviving = rest[st.upper[rest] - eps >= threshold]
        st.active = np.concatenate([prefix, surviving])
    else:
        st.active = prefix
    if st.active.size > k:
        return False
    if prefix.size >= 2:
        return bool((st.upper[prefix[1:]] - eps < st.lower[prefix[:-1]]).all())
    return True


def check_converged_reference(st: OracleState) -> bool:
    """engine.py:333-379 exactly as the reference computes it (argpartition
    for the cut, engine.py:359) -- the CPU *baseline* path, timed by
    bench.py.  check_converged above is the checker's variant (the device's
    deterministic tie rule); both give the same verdicts, thresholds and
    prefixes whenever no exact tie straddles the k-th position (SURVEY.md
    8(c) rule 4), as on every R-MAT config."""
    kind = st.crit.kind
    eps = st.epsilon
    if kind in (SCORE, PAIR):
        return check_converged(st)
    k = st.n if kind == RANKING else st.crit.k
    m = st.active
    lowers = st.lower[m]
    if m.size > k:
        sel = np.argpartition(-lowers, k - 1)
        top_pos, rest_pos = sel[:k], sel[k:]
    else:
        top_pos = np.arange(m.size)
        rest_pos = np.empty(0, dtype=np.int64)
    top_ids = m[top_pos]
    prefix = top_ids[np.lexsort((top_ids, -st.lower[top_ids]))]
    threshold = st.lower[prefix[-1]]
    if rest_pos.size:
        rest = m[rest_pos]
        st.active = np.concatenate([prefix, rest[st.upper[rest] - eps >= threshold]])
    else:
        st.active = prefix
    if st.active.size > k:
        return False
    if prefix.size >= 2:
        return bool((st.upper[prefix[1:]] - eps < st.lower[prefix[:-1]]).all())
    return True


def run_reference_path(st: OracleState, g: CSRGraph) -> "OracleResult":
    """engine.run (engine.py:382-396) with the reference's own check: the
    timed CPU baseline (bench.py --impl reference and cpu_baseline)."""
    while True:
        iterate_once(st, g)
        if check_converged_reference(st):
            break
        if st.r >= st.max_iterations:
            raise OracleConvergenceError(st.r, st.gap())
    return ranking_result(st)


class OracleConvergenceError(Exception):
    def __init__(self, iterations, gap):
        super().__init__(f"unmet after {iterations} iterations")
        self.iterations = iterations
        self.gap = gap


@dataclass
class OracleResult:
    order: np.ndarray
    lower: np.ndarray
    upper: np.ndarray
    iterations_used: int
    separated_fraction: float
    separated_pairs: int = 0

    def top(self, k: int) -> list[int]:
        return [int(v) for v in self.order[:k]]


def run(st: OracleState, g: CSRGraph) -> OracleResult:
    """engine.py:382-396."""
    while True:
        iterate_once(st, g)
        if check_converged(st):
            break
        if st.r >= st.max_iterations:
            raise OracleConvergenceError(st.r, st.gap())
    return ranking_result(st)


def separated_pairs(lower: np.ndarray, upper: np.ndarray) -> int:
    """engine.py:420-426: sum_v #{w : lower[w] > upper[v]} as an exact int."""
    n = lower.size
    sorted_lower = np.sort(lower)
    above = n - np.searchsorted(sorted_lower, upper, side="right")
    return int(above.sum())


def separated_fraction(st: OracleState) -> float:
    """engine.py:411-427."""
    n = st.n
    if n < 2:
        return 1.0
    return separated_pairs(st.lower, st.upper) / (n * (n - 1) // 2)


def ranking_result(st: OracleState) -> OracleResult:
    """engine.py:399-408."""
    order = np.lexsort((np.arange(st.n), -st.lower))
    n = st.n
    pairs = separated_pairs(st.lower, st.upper) if n >= 2 else 0
    frac = 1.0 if n < 2 else pairs / (n * (n - 1) // 2)
    return OracleResult(order, st.lower.copy(), st.upper.copy(), st.r, frac,
                        pairs)


# ---------------------------------------------------------------- dynamic

@dataclass
class OracleUpdateStats:
    """UpdateStats (dynamic.py:28-38)."""
    batch_size: int = 0
    seeds: int = 0
    visited: int = 0
    level_sizes: list = field(default_factory=list)
    reactivated: int = 0
    aborted_level: int | None = None
    resumed_iterations: int = 0


class AdjGraph(CSRGraph):
    """Mutable set-of-sets graph for the dynamic oracle (graph.py:80-255)."""

    def __init__(self, n: int, arcs=()):
        self.node_count = n
        self._out = [set() for _ in range(n)]
        self._in = [set() for _ in range(n)]
        for u, v in arcs:
            self._out[u].add(v)
            self._in[v].add(u)
        self.version = 1
        self._sym = None
        self._csr = None
        self._rebuild()

    @classmethod
    def from_csr(cls, g: CSRGraph) -> "AdjGraph":
        rows = np.repeat(np.arange(g.node_count), np.diff(g.indptr))
        return cls(g.node_count, zip(rows.tolist(), g.indices.tolist()))

    def _rebuild(self):
        n = self.node_count
        indptr = np.zeros(n + 1, dtype=np.int64)
        indptr[1:] = np.cumsum([len(s) for s in self._out])
        indices = np.empty(int(indptr[-1]), dtype=np.int32)
        for v in range(n):
            indices[indptr[v]:indptr[v + 1]] = sorted(self._out[v])
        self.indptr, self.indices = indptr, indices
        self._sym = None
        self._csr = None

    def in_neighbors(self, v):
        return iter(self._in[v])

    def has_arc(self, u, v):
        return v in self._out[u]

    def remove_arcs(self, arcs):
        for u, v in arcs:
            self._out[u].discard(v)
            self._in[v].discard(u)
        self.version += 1
        self._rebuild()

    def insert_arcs(self, arcs):
        for u, v in arcs:
            self._out[u].add(v)
            self._in[v].add(u)
        self.version += 1
        self._rebuild()


def update_batch(st: OracleState, g: AdjGraph, insertions, deletions,
                 theta: float = 0.5) -> OracleUpdateStats:
    """dynamic.py:126-211 with update_level (dynamic.py:63-123) inlined.

    Validation (dynamic.py:137-161) is left to the caller; this restates the
    numeric path: deletions, per-level repair, bound refresh, reactivation,
    insertions, resume.
    """
    alpha = st.alpha
    ins = [(int(a), int(b)) for a, b in insertions]
    dels = [(int(a), int(b)) for a, b in deletions]
    degs = g.out_degrees().copy()
    for s, _ in dels:
        degs[s] -= 1
    for s, _ in ins:
        degs[s] += 1
    new_max = int(degs.max()) if st.n else 0
    stats = OracleUpdateStats(batch_size=len(ins) + len(dels))
    seeds = {s for s, _ in ins} | {s for s, _ in dels}
    targets = {t for _, t in ins} | {t for _, t in dels}
    stats.seeds = len(seeds)
    affected = set(seeds)
    old_prev: dict = {}
    aborted = False
    g.remove_arcs(dels)
    for level in range(1, st.r + 1):
        w_prev = st.levels[level - 1]
        w_cur = st.levels[level]
        if aborted or len(affected) > theta * st.n:        # dynamic.py:78
            if not aborted:
                aborted = True
                stats.aborted_level = level
            new = alpha * csr_matvec(g, w_prev, st.threads)
            for s, t in ins:
                new[s] += alpha * w_prev[t]
            st.katz += new - w_cur
            st.levels[level] = new
            old_prev = {}
            continue
        stats.level_sizes.append(len(affected))
        old_cur: dict = {}
        for v in list(affected):                          # dynamic.py:94-103
            old = old_prev.get(v)
            if old is None or old == w_prev[v]:
                continue
            push = alpha * (w_prev[v] - old)
            for w in g.in_neighbors(v):
                affected.add(w)
                if w not in old_cur:
                    old_cur[w] = float(w_cur[w])
                w_cur[w] += push
        for s, t in ins:                                  # :107-110
            if s not in old_cur:
                old_cur[s] = float(w_cur[s])
            w_cur[s] += alpha * w_prev[t]
        for s, t in dels:                                 # :111-117
            base = old_prev.get(t)
            if base is None:
                base = float(w_prev[t])
            if s not in old_cur:
                old_cur[s] = float(w_cur[s])
            w_cur[s] -= alpha * base
        for w, old in old_cur.items():                    # :120-121
            st.katz[w] += w_cur[w] - old
        old_prev = old_cur
    stats.visited = len(affected | targets)
    st.gamma = tail_gamma(alpha, new_max)                 # :181-187
    tail = alpha * st.levels[st.r]
    st.lower = st.katz + tail if st.undirected else st.katz.copy()
    st.upper = st.katz + tail * st.gamma
    if st.crit.kind in (RANKING, TOPK) and st.active.size < st.n:  # :190-197
        floor = float(np.min(st.lower[st.active])) - st.epsilon
        inactive = np.setdiff1d(np.arange(st.n, dtype=np.int64), st.active)
        back = inactive[st.upper[inactive] >= floor]
        if back.size:
            st.active = np.concatenate([st.active, back])
            stats.reactivated = int(back.size)
    g.insert_arcs(ins)
    while not check_converged(st):                        # :203-210
        if st.r >= st.max_iterations:
            st.last_update_stats = stats
            raise OracleConvergenceError(st.r, st.gap())
        iterate_once(st, g)
        stats.resumed_iterations += 1
    st.last_update_stats = stats
    return stats


# ---------------------------------------------------------------- baselines
# Restatement of baselines.py:36-154 and cli.py:349-386 (the paper's
# comparison methods and the ranking-agreement measure).

class OracleBaselineError(Exception):
    """kind: 'convergence' | 'numeric' | 'not_applicable' | 'parameter'."""

    def __init__(self, kind, partial=None, iterations=None):
        super().__init__(kind)
        self.kind, self.partial, self.iterations = kind, partial, iterations


@dataclass
class OracleScores:
    method: str
    values: np.ndarray
    iterations: int | None = None
    residual: float | None = None

    def ranking(self) -> np.ndarray:                       # baselines.py:30-33
        n = len(self.values)
        return np.lexsort((np.arange(n), -self.values))


def _baseline_alpha(g: CSRGraph, alpha):
    d = g.max_out_degree()
    if alpha is None:
        alpha = default_alpha(d)                            # engine.py:96-99
    if alpha <= 0 or (d > 0 and alpha >= 1.0 / d) or (d == 0 and alpha >= 1.0):
        raise OracleBaselineError("parameter")              # engine.py:102-113
    return alpha


def foster(g: CSRGraph, alpha=None, tol=1e-9, max_iter=1000) -> OracleScores:
    """baselines.py:36-68: c <- alpha*A*c + 1 until max|change| < tol."""
    alpha = _baseline_alpha(g, alpha)
    if not tol > 0 or max_iter < 1:
        raise OracleBaselineError("parameter")
    c = np.ones(g.node_count, dtype=np.float64)
    delta = np.inf
    for it in range(1, max_iter + 1):
        nxt = alpha * csr_matvec(g, c) + 1.0                # :58
        delta = float(np.max(np.abs(nxt - c))) if len(c) else 0.0
        c = nxt
        if delta < tol:
            return OracleScores("foster", c - 1.0, iterations=it, residual=delta)
    raise OracleBaselineError("convergence",
                              OracleScores("foster", c - 1.0, max_iter, delta), max_iter)


def cg_katz(g: CSRGraph, alpha=None, residual_tol=1e-15, max_iter=None) -> OracleScores:
    """baselines.py:71-129: plain CG on (I - alpha*A) z = 1 from z = 1."""
    alpha = _baseline_alpha(g, alpha)
    if not residual_tol > 0:
        raise OracleBaselineError("parameter")
    if not g.is_symmetric():
        raise OracleBaselineError("not_applicable")
    n = g.node_count
    if max_iter is None:
        max_iter = 10 * n + 100

    def system(v):
        return v - alpha * csr_matvec(g, v)

    b = np.ones(n)
    x = np.ones(n)
    r = b - system(x)
    rs = float(r @ r)
    it = 0
    if np.sqrt(rs) >= residual_tol:
        p = r.copy()
        while it < max_iter:
            Ap = system(p)
            denom = float(p @ Ap)
            if denom <= 0.0 or not np.isfinite(denom):
                raise OracleBaselineError("numeric")
            step = rs / denom
            x += step * p
            r -= step * Ap
            rs_next = float(r @ r)
            it += 1
            if np.sqrt(rs_next) < residual_tol:
                rs = rs_next
                break
            p = r + (rs_next / rs) * p
            rs = rs_next
        else:
            raise OracleBaselineError(
                "convergence", OracleScores("cg", alpha * csr_matvec(g, x), it,
                                            float(np.sqrt(rs))), it)
    return OracleScores("cg", alpha * csr_matvec(g, x), iterations=it,
                        residual=float(np.sqrt(rs)))


def dense_oracle(g: CSRGraph, alpha=None) -> OracleScores:
    """baselines.py:132-154: LU solve of (I - alpha*A) z = 1; alpha*A*z."""
    if g.node_count > 2000:
        raise OracleBaselineError("parameter")
    alpha = _baseline_alpha(g, alpha)
    A = np.zeros((g.node_count, g.node_count))
    for v in range(g.node_count):
        A[v, g.indices[g.indptr[v]:g.indptr[v + 1]]] = 1.0
    z = np.linalg.solve(np.eye(g.node_count) - alpha * A, np.ones(g.node_count))
    return OracleScores("dense", alpha * (A @ z))


def inversions(seq: np.ndarray) -> int:
    """Pairs i < j with seq[i] > seq[j] (cli.py:363-386 counts the same by
    merge sort); here a Fenwick tree over the values 0..n-1."""
    seq = np.asarray(seq, dtype=np.int64)
    n = seq.size
    tree = np.zeros(n + 1, dtype=np.int64)
    inv = 0
    for i in range(n - 1, -1, -1):           # count smaller values to the right
        j = int(seq[i])
        while j > 0:
            inv += int(tree[j])
            j -= j & -j
        j = int(seq[i]) + 1
        while j <= n:
            tree[j] += 1
            j += j & -j
    return inv


def concordant_fraction(order_a, order_b) -> float:
    """cli.py:349-360."""
    n = len(order_a)
    if n < 2:
        return 1.0
    pos = np.empty(n, dtype=np.int64)
    pos[np.asarray(order_a)] = np.arange(n)
    seq = pos[np.asarray(order_b)]
    return 1.0 - inversions(seq) / (n * (n - 1) // 2)
