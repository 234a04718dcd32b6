"""Bounded-Katz engine: the reference's Python surface over the B200 kernels.

Mirrors katzbounds.engine (/root/reference/pkg/src/katzbounds/engine.py) --
same names, argument meaning, defaults and errors -- while the state lives
on the device and every numeric step runs in the native library
(include/katzb200.h):

  iterate_once   -> kb_iterate   (K1 fused SpMV + bounds, engine.py:296-319)
  check_converged-> kb_check     (K2 device selection/sort, :333-379)
  run            -> kb_run       (device loop, :382-396) + ranking_result
  ranking_result -> kb_result    (K3 device sort + separated pairs, :399-427)

Parameters (alpha, gamma, the iteration cap) are computed here with the
reference's own expressions so the kernels receive bit-identical inputs.
There is no CPU path: without the library or a GPU these calls raise.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import FrozenInstanceError, dataclass, replace

import numpy as np

from . import _lib
from .errors import ConvergenceError, ParameterError, StateError
from .graph import csr_of

DEFAULT_EPSILON = 1e-6

RANKING = "ranking"
TOPK = "topk"
SCORE = "score"
PAIR = "pair"

_KIND = {RANKING: _lib.KB_RANKING, TOPK: _lib.KB_TOPK, SCORE: _lib.KB_SCORE,
         PAIR: _lib.KB_PAIR}


# ---------------------------------------------------------------- criteria

@dataclass(frozen=True)
class Criterion:
    """Stopping rule (engine.py:36-83): ranking / topk / score / pair."""

    kind: str
    epsilon: float = DEFAULT_EPSILON
    k: int | None = None
    u: int | None = None
    v: int | None = None

    def __post_init__(self):
        if self.kind not in (RANKING, TOPK, SCORE, PAIR):
            raise ParameterError(f"unknown criterion kind {self.kind!r}")
        if not (isinstance(self.epsilon, (int, float)) and
                math.isfinite(self.epsilon) and self.epsilon > 0):
            raise ParameterError(f"epsilon must be finite and > 0, got {self.epsilon}")
        if self.kind == TOPK:
            if self.k is None or int(self.k) < 1:
                raise ParameterError("topk criterion needs k >= 1")
        if self.kind == PAIR:
            if self.u is None or self.v is None:
                raise ParameterError("pair criterion needs two node ids")
            if self.u == self.v:
                raise ParameterError("pair criterion needs two distinct nodes")
            if self.u < 0 or self.v < 0:
                raise ParameterError("pair node ids must be non-negative")

    @classmethod
    def ranking(cls, epsilon: float = DEFAULT_EPSILON) -> "Criterion":
        return cls(RANKING, epsilon)

    @classmethod
    def top_k(cls, k: int, epsilon: float = DEFAULT_EPSILON) -> "Criterion":
        return cls(TOPK, epsilon, k=int(k))

    @classmethod
    def score(cls, epsilon: float = DEFAULT_EPSILON) -> "Criterion":
        return cls(SCORE, epsilon)

    @classmethod
    def pair(cls, u: int, v: int, epsilon: float = DEFAULT_EPSILON) -> "Criterion":
        return cls(PAIR, epsilon, u=int(u), v=int(v))


@dataclass(frozen=True)
class Params:
    """engine.py:86-93."""

    alpha: float
    epsilon: float
    gamma: float
    keep_all_levels: bool = True


def default_alpha(g) -> float:
    """1 / (1 + max out-degree); 0.5 on an edgeless graph (engine.py:96-99)."""
    d = g.max_out_degree()
    return 1.0 / (1.0 + d) if d > 0 else 0.5


def validate_alpha(alpha: float, max_out_degree: int) -> None:
    """engine.py:102-113."""
    if not (isinstance(alpha, (int, float)) and math.isfinite(alpha)):
        raise ParameterError(f"alpha must be a finite number, got {alpha!r}")
    if alpha <= 0.0:
        raise ParameterError(f"alpha must be > 0, got {alpha}")
    if max_out_degree > 0:
        if alpha >= 1.0 / max_out_degree:
            raise ParameterError(
                f"alpha={alpha} is not below 1/max_out_degree = "
                f"1/{max_out_degree}; the walk series may diverge")
    elif alpha >= 1.0:
        raise ParameterError(f"alpha must be < 1, got {alpha}")


def tail_gamma(alpha: float, max_out_degree: int) -> float:
    """deg_max / (1 - alpha * deg_max); 0 if edgeless (engine.py:116-119)."""
    d = max_out_degree
    return d / (1.0 - alpha * d) if d > 0 else 0.0


def default_iteration_cap(alpha: float, max_out_degree: int, epsilon: float) -> int:
    """10 * ceil(log(1/eps) / log(1/(alpha*deg_max))) (engine.py:286-293)."""
    rho = alpha * max_out_degree
    if rho <= 0.0:
        return 64
    cap = 10 * math.ceil(math.log(1.0 / epsilon) / math.log(1.0 / rho))
    return max(1, cap)


# ---------------------------------------------------------------- device graph

class DeviceGraph:
    """A kb_graph handle: the device SELL layout of one graph version."""

    def __init__(self, indptr: np.ndarray, indices: np.ndarray, *, device: int = 0,
                 split_threshold: int = 0, hot_size: int = -1):
        L = _lib.lib()
        indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        indices = np.ascontiguousarray(indices, dtype=np.int32)
        n = indptr.size - 1
        h = ctypes.c_void_p()
        _lib.check(L.kb_graph_create(device, n, int(indptr[-1]), _lib.ptr(indptr),
                                     _lib.ptr(indices), split_threshold, hot_size,
                                     ctypes.byref(h)))
        self._h = h
        self.device = device
        self._L = L

    @property
    def handle(self):
        return self._h

    def info(self) -> _lib.GraphInfo:
        info = _lib.GraphInfo()
        _lib.check(self._L.kb_graph_info_get(self._h, ctypes.byref(info)))
        return info

    def is_symmetric(self) -> bool:
        out = ctypes.c_int()
        _lib.check(self._L.kb_graph_is_symmetric(self._h, ctypes.byref(out)))
        return bool(out.value)

    def close(self):
        if getattr(self, "_h", None):
            self._L.kb_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_FOREIGN_CACHE: list = []   # [(graph, version, DeviceGraph)] for foreign graph types


def device_graph(g, device: int = 0) -> DeviceGraph:
    """The device copy of g at its current version (uploaded on first use)."""
    cached = getattr(g, "_device", None) if hasattr(g, "_device") else None
    if cached is not None and cached[0] == g.version and cached[1].device == device:
        return cached[1]
    if not hasattr(g, "_device"):
        for ent in _FOREIGN_CACHE:
            if ent[0] is g and ent[1] == g.version and ent[2].device == device:
                return ent[2]
    indptr, indices = csr_of(g)
    dg = DeviceGraph(indptr, indices, device=device)
    if hasattr(g, "_device"):
        g._device = (g.version, dg)
    else:
        _FOREIGN_CACHE.insert(0, (g, g.version, dg))
        del _FOREIGN_CACHE[4:]
    return dg


# ---------------------------------------------------------------- state

class _Levels:
    """Read-only list view of KatzState.levels (engine.py:147, :317)."""

    def __init__(self, st: "KatzState"):
        self._st = st

    def __len__(self) -> int:
        return self._st._info().levels_kept

    def __getitem__(self, i):
        n = len(self)
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(n))]
        if i < 0:
            i += n
        if not 0 <= i < n:
            raise IndexError("level index out of range")
        base = self._st.r + 1 - n
        return self._st._vector(_lib.KB_VEC_LEVEL, base + i)

    def __iter__(self):
        for i in range(len(self)):
            yield self[i]


class KatzState:
    """Device-resident state of one bounded-Katz computation.

    Attribute surface of engine.py:124-177: n, params, criterion,
    undirected, r, levels, katz, lower, upper, active, graph_version,
    threads, max_iterations (assignable), last_update_stats, alpha, gamma,
    epsilon, gap().  Vectors are fetched from the device on access (by node
    id, read-only numpy arrays).
    """

    def __init__(self, dg: DeviceGraph, n: int, params: Params, criterion: Criterion,
                 undirected: bool, graph_version: int, threads: int, max_iterations: int):
        self.n = n
        self.params = params
        self.criterion = criterion
        self.undirected = undirected
        self.graph_version = graph_version
        self.threads = threads
        self.last_update_stats = None
        self._dg = dg
        self._L = _lib.lib()
        c = criterion
        h = ctypes.c_void_p()
        _lib.check(self._L.kb_state_create(
            dg.handle, params.alpha, params.gamma, int(undirected), _KIND[c.kind],
            c.epsilon, int(c.k or 0), int(c.u or 0), int(c.v or 0),
            int(params.keep_all_levels), int(max_iterations), ctypes.byref(h)))
        self._h = h
        self._tick = 0
        self._cache: dict = {}

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                self._L.kb_state_destroy(self._h)
                self._h = None
        except Exception:
            pass

    # -- bookkeeping
    def _touch(self):
        self._tick += 1
        self._cache.clear()

    def _info(self) -> _lib.StateInfo:
        info = _lib.StateInfo()
        _lib.check(self._L.kb_state_info_get(self._h, ctypes.byref(info)))
        return info

    def _vector(self, which: int, level: int = 0) -> np.ndarray:
        key = (which, level)
        a = self._cache.get(key)
        if a is None:
            a = np.empty(self.n, dtype=np.float64)
            _lib.check(self._L.kb_get_vector(self._h, which, level, _lib.ptr(a)))
            a.setflags(write=False)
            self._cache[key] = a
        return a

    # -- reference attributes
    @property
    def r(self) -> int:
        return int(self._info().r)

    @property
    def alpha(self) -> float:
        return self.params.alpha

    @property
    def gamma(self) -> float:
        return self.params.gamma

    @property
    def epsilon(self) -> float:
        return self.criterion.epsilon

    @property
    def max_iterations(self) -> int:
        return int(self._info().max_iterations)

    @max_iterations.setter
    def max_iterations(self, value: int) -> None:
        _lib.check(self._L.kb_state_set_max_iterations(self._h, int(value)))

    @property
    def levels(self) -> _Levels:
        return _Levels(self)

    @property
    def katz(self) -> np.ndarray:
        return self._vector(_lib.KB_VEC_KATZ)

    @property
    def lower(self) -> np.ndarray:
        return self._vector(_lib.KB_VEC_LOWER)

    @property
    def upper(self) -> np.ndarray:
        return self._vector(_lib.KB_VEC_UPPER)

    @property
    def active(self) -> np.ndarray:
        a = self._cache.get("active")
        if a is None:
            m = int(self._info().active)
            a = np.empty(m, dtype=np.int64)
            if m:
                _lib.check(self._L.kb_get_active(self._h, _lib.ptr(a)))
            a.setflags(write=False)
            self._cache["active"] = a
        return a

    @property
    def k_boundary_ties(self) -> int:
        """SURVEY.md 8(c) rule 4: nodes that tied the k-th lower bound exactly
        and were dropped from the active set with gap < eps, summed over this
        state's TOPK checks.  The reference's argpartition (engine.py:359)
        picks among such ties arbitrarily, so while this is 0 the active set
        and r are the reference's whatever its choice; otherwise run() warns
        (KBoundaryTieWarning) that they may differ (the certified order and
        the bounds never do: ranking_result sorts every node)."""
        return int(self._info().k_boundary_ties)

    def gap(self) -> float:
        """Widest remaining bound interval (engine.py:172-174)."""
        out = ctypes.c_double()
        _lib.check(self._L.kb_gap(self._h, ctypes.byref(out)))
        return float(out.value)

    def set_gamma(self, gamma: float) -> None:
        self.params = replace(self.params, gamma=gamma)

    @property
    def device_graph(self) -> DeviceGraph:
        return self._dg


# ---------------------------------------------------------------- results

class _DeviceRanking:
    """A kb_ranking snapshot: the ranked vectors left in HBM until read."""

    def __init__(self, h, n: int):
        self._h, self.n, self._L = h, n, _lib.lib()

    def read(self, which: int, start: int, stop: int) -> np.ndarray:
        out = np.empty(max(0, stop - start), dtype=np.int64 if which == 0 else np.float64)
        if out.size:
            _lib.check(self._L.kb_ranking_read(self._h, which, start, out.size, _lib.ptr(out)))
        return out

    def __del__(self):
        try:
            if self._h:
                self._L.kb_ranking_destroy(self._h)
                self._h = None
        except Exception:
            pass


class RankingResult:
    """Immutable outcome of a converged run (engine.py:224-243).

    Same fields and methods as the reference's frozen dataclass.  A result
    made by ranking_result keeps its vectors on the device and copies each
    one to the host the first time it is touched; ``top(k)`` and
    ``bounds(v)`` copy only what they return.  Materialised arrays are
    read-only, as in the reference."""

    __slots__ = ("_order", "_lower", "_upper", "iterations_used", "criterion",
                 "separated_fraction", "_dev")

    def __init__(self, order=None, lower=None, upper=None, iterations_used: int = 0,
                 criterion: Criterion | None = None, separated_fraction: float = 0.0, *,
                 _device: _DeviceRanking | None = None):
        set_ = object.__setattr__
        set_(self, "_order", order)
        set_(self, "_lower", lower)
        set_(self, "_upper", upper)
        set_(self, "iterations_used", iterations_used)
        set_(self, "criterion", criterion)
        set_(self, "separated_fraction", separated_fraction)
        set_(self, "_dev", _device)

    def __setattr__(self, name, value):
        raise FrozenInstanceError(f"cannot assign to field {name!r}")

    def __delattr__(self, name):
        raise FrozenInstanceError(f"cannot delete field {name!r}")

    def _field(self, slot: str, which: int) -> np.ndarray:
        arr = object.__getattribute__(self, slot)
        if arr is None:
            dev = self._dev
            arr = dev.read(which, 0, dev.n)
            arr.setflags(write=False)
            object.__setattr__(self, slot, arr)
            if all(object.__getattribute__(self, x) is not None
                   for x in ("_order", "_lower", "_upper")):
                object.__setattr__(self, "_dev", None)   # all on the host: free HBM
        return arr

    @property
    def order(self) -> np.ndarray:
        return self._field("_order", 0)

    @property
    def lower(self) -> np.ndarray:
        return self._field("_lower", 1)

    @property
    def upper(self) -> np.ndarray:
        return self._field("_upper", 2)

    def bounds(self, v: int) -> tuple[float, float]:
        if self._lower is None and self._dev is not None:
            v = int(v)
            if not -self._dev.n <= v < self._dev.n:
                raise IndexError(f"index {v} is out of bounds for axis 0 with size {self._dev.n}")
            v %= self._dev.n
            return (float(self._dev.read(1, v, v + 1)[0]), float(self._dev.read(2, v, v + 1)[0]))
        return float(self.lower[v]), float(self.upper[v])

    def top(self, k: int) -> list[int]:
        if self._order is None and self._dev is not None:
            n = self._dev.n
            stop = max(0, min(int(k), n)) if k >= 0 else max(0, n + int(k))
            return [int(v) for v in self._dev.read(0, 0, stop)]
        return [int(v) for v in self.order[:k]]

    def __repr__(self) -> str:
        return (f"RankingResult(iterations_used={self.iterations_used}, "
                f"criterion={self.criterion!r}, separated_fraction={self.separated_fraction!r})")


# ---------------------------------------------------------------- operations

# Graph.is_symmetric on the host sorts every arc key (~12 s at C2); a large
# graph is uploaded here anyway, and the pipelined ingest decides the same
# question while its arcs stream in (kb_graph_is_symmetric).  Small graphs
# keep the host test, so bad arguments are still rejected before any device
# work.
_HOST_SYMMETRY_ARCS = 1 << 22


def _symmetric(g, device: int) -> bool:
    arcs = getattr(g, "arc_count", None)
    if arcs is None or arcs <= _HOST_SYMMETRY_ARCS:
        return bool(g.is_symmetric())
    return device_graph(g, device).is_symmetric()


def init(g, criterion: Criterion, *, alpha: float | None = None,
         undirected: bool = False, keep_all_levels: bool = True,
         threads: int = 1, max_iterations: int | None = None,
         device: int = 0) -> KatzState:
    """engine.py:248-283; the graph is uploaded to `device` (cached per version).

    `threads` is validated and recorded for API compatibility; the device
    parallelism does not depend on it (results are identical for any value,
    as in the reference, engine.py:184-187).
    """
    n = g.node_count
    if n < 1:
        raise ParameterError("graph must have at least one node")
    if alpha is None:
        alpha = default_alpha(g)
    alpha = float(alpha)
    d = g.max_out_degree()
    validate_alpha(alpha, d)
    if criterion.kind == TOPK and criterion.k > n:
        raise ParameterError(f"topk k={criterion.k} exceeds node count {n}")
    if criterion.kind == PAIR and (criterion.u >= n or criterion.v >= n):
        raise ParameterError("pair criterion names a node outside the graph")
    if undirected and not _symmetric(g, device):
        raise ParameterError("undirected mode requires a symmetric arc set")
    if threads < 1:
        raise ParameterError(f"threads must be >= 1, got {threads}")
    gamma = tail_gamma(alpha, d)
    if max_iterations is None:
        max_iterations = default_iteration_cap(alpha, d, criterion.epsilon)
    elif max_iterations < 1:
        raise ParameterError("max_iterations must be >= 1")
    params = Params(alpha=alpha, epsilon=criterion.epsilon, gamma=gamma,
                    keep_all_levels=keep_all_levels)
    dg = device_graph(g, device)
    return KatzState(dg, n, params, criterion, undirected, g.version, int(threads),
                     int(max_iterations))


def _check_graph(state: KatzState, g) -> None:
    if g.version != state.graph_version:
        raise StateError("graph changed since init; static iteration would be unsound")


def iterate_once(state: KatzState, g) -> None:
    """Advance one walk level and refresh every bound (engine.py:296-319)."""
    _check_graph(state, g)
    state._touch()
    _lib.check(state._L.kb_iterate(state._h, 1))


def epsilon_separated(state: KatzState, w: int, v: int) -> bool:
    """lower(w) > upper(v) - eps (engine.py:322-330)."""
    for x in (w, v):
        if not 0 <= x < state.n:
            raise ParameterError(f"node id {x} outside graph")
    out = ctypes.c_int()
    _lib.check(state._L.kb_epsilon_separated(state._h, int(w), int(v), ctypes.byref(out)))
    return bool(out.value)


def check_converged(state: KatzState) -> bool:
    """Evaluate the stopping rule on the device (engine.py:333-379)."""
    state._touch()
    out = ctypes.c_int()
    _lib.check(state._L.kb_check(state._h, ctypes.byref(out)))
    return bool(out.value)


def run(state: KatzState, g) -> RankingResult:
    """Iterate until the stopping rule holds; error out at the cap
    (engine.py:382-396).  The loop runs inside the native library."""
    _check_graph(state, g)
    state._touch()
    out = ctypes.c_int()
    st = state._L.kb_run(state._h, ctypes.byref(out))
    if st == _lib.KB_ECONVERGENCE:
        msg = _lib.last_error()
        raise ConvergenceError(msg, iterations=state.r, gap=state.gap())
    _lib.check(st)
    if state.criterion.kind == TOPK:
        ties = state.k_boundary_ties
        if ties:
            import warnings
            warnings.warn(KBoundaryTieWarning(
                f"{ties} node(s) tied the k-th lower bound exactly and were dropped with "
                f"gap < epsilon: the reference's argpartition may keep a different active "
                f"set (SURVEY.md 8(c) rule 4)"), stacklevel=2)
    return ranking_result(state)


class KBoundaryTieWarning(UserWarning):
    """An exact tie at the k-th position was resolved by node id where the
    reference's np.argpartition (engine.py:359) resolves it arbitrarily."""


def ranking_result(state: KatzState) -> RankingResult:
    """Snapshot the bounds into an immutable ranking (engine.py:399-408)."""
    n = state.n
    if state.r < 1:
        raise StateError("separated_fraction needs at least one iteration")
    pairs = ctypes.c_int64()
    h = ctypes.c_void_p()
    _lib.check(state._L.kb_ranking_snapshot(state._h, ctypes.byref(h), ctypes.byref(pairs)))
    frac = 1.0 if n < 2 else int(pairs.value) / (n * (n - 1) // 2)
    return RankingResult(iterations_used=state.r, criterion=state.criterion,
                         separated_fraction=frac, _device=_DeviceRanking(h, n))


def separated_fraction(state: KatzState) -> float:
    """Fraction of unordered pairs strictly separated (engine.py:411-427)."""
    if state.r < 1:
        raise StateError("separated_fraction needs at least one iteration")
    n = state.n
    if n < 2:
        return 1.0
    pairs = ctypes.c_int64()
    _lib.check(state._L.kb_separated_pairs(state._h, ctypes.byref(pairs)))
    return int(pairs.value) / (n * (n - 1) // 2)
