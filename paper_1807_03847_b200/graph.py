"""Host graph store with the reference's Graph/EdgeBatch surface.

Mirrors katzbounds.graph (/root/reference/pkg/src/katzbounds/graph.py:30-255)
-- same methods, argument meaning and errors -- but stores the arc set as a
sorted array of packed keys ``u * n + v`` instead of Python set-of-sets, so
graphs with hundreds of millions of arcs fit in memory and build in seconds.
The canonical CSR (rows ascending, graph.py:177-197) is derived from that
array per version and is what the device ingest (``kb_graph_create``) reads.

Any object with the reference's duck-typed surface (node_count, version,
max_out_degree(), is_symmetric(), out_csr()) -- including a real
``katzbounds.Graph`` -- is accepted by the engine as well.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Iterable, Iterator, Sequence

import itertools

import numpy as np

from .errors import BatchPreconditionError, NodeRangeError

Arc = tuple[int, int]
MAX_NODE_ID = 2**31 - 1   # graph.py:27


def check_batch_arcs(batch: "EdgeBatch", n: int, check_node, present) -> None:
    """The per-arc checks of Graph.validate_batch (graph.py:207-220) in the
    reference's order -- insertions, then deletions; per arc, the range of
    u, of v, then presence -- vectorised: the first arc that fails any test
    raises that test's error.  present((m, 2) int64 in-range arcs) -> bool[m]."""
    try:
        arrays = batch.arrays()
    except OverflowError:
        arrays = None
    if arrays is None:              # ids beyond int64: the exact per-arc path
        for u, v in batch.insertions + batch.deletions:
            check_node(u)
            check_node(v)
        return
    for a, arcs, want, msg in ((arrays[0], batch.insertions, False, "already present"),
                               (arrays[1], batch.deletions, True, "not present")):
        if not a.shape[0]:
            continue
        if a.min() >= 0 and a.max() < n:        # the common case: no range fault
            fault = present(np.ascontiguousarray(a)) != want
            if fault.any():
                i = int(np.argmax(fault))
                u, v = arcs[i]
                verb = "insert" if not want else "delete"
                raise BatchPreconditionError(f"cannot {verb} arc ({u}, {v}): {msg}")
            continue
        bad = ((a < 0) | (a >= n)).any(axis=1)
        fault = bad.copy()
        ok = ~bad
        if ok.any():
            fault[ok] = present(np.ascontiguousarray(a[ok])) != want
        if fault.any():
            i = int(np.argmax(fault))
            u, v = arcs[i]
            if bad[i]:
                check_node(u)
                check_node(v)
            verb = "insert" if not want else "delete"
            raise BatchPreconditionError(f"cannot {verb} arc ({u}, {v}): {msg}")


class ArcArray(Sequence):
    """An (m, 2) int64 arc array with the read-only list-of-tuples surface
    EdgeBatch exposes (len, index, iterate, compare, concatenate): large
    batches built from numpy arrays never become Python tuples unless a
    caller walks them."""

    def __init__(self, a: np.ndarray):
        self.a = a

    def __len__(self) -> int:
        return self.a.shape[0]

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [tuple(x) for x in self.a[i].tolist()]
        u, v = self.a[i].tolist()
        return (u, v)

    def __iter__(self):
        return iter(tuple(x) for x in self.a.tolist())

    def __eq__(self, other) -> bool:
        return list(self) == list(other)

    def __add__(self, other):
        return list(self) + list(other)

    def __radd__(self, other):
        return list(other) + list(self)

    def __repr__(self) -> str:
        return repr(list(self))


def _arcs_in(x):
    if isinstance(x, ArcArray):
        return x
    if isinstance(x, np.ndarray):
        a = np.ascontiguousarray(x, dtype=np.int64)
        if a.size == 0:
            a = a.reshape(0, 2)
        if a.ndim != 2 or a.shape[1] != 2:
            raise ValueError("arc arrays must have shape (m, 2)")
        if x.dtype != np.int64 and not np.array_equal(a, x):
            raise ValueError("arc ids must be integers")
        return ArcArray(a)
    return [(int(u), int(v)) for u, v in x]


@dataclass
class EdgeBatch:
    """Arc insertions and deletions applied as one unit (graph.py:30-68).

    Besides lists of (u, v) pairs, either side may be an (m, 2) integer
    numpy array (kept as an array: no per-arc Python objects)."""

    insertions: list[Arc] = field(default_factory=list)
    deletions: list[Arc] = field(default_factory=list)

    def __post_init__(self):
        self.insertions = _arcs_in(self.insertions)
        self.deletions = _arcs_in(self.deletions)

    def arrays(self) -> tuple[np.ndarray, np.ndarray]:
        """(insertions, deletions) as (m, 2) int64 arrays: an array side as
        is, a list side converted once per list object and length (the lists
        are the batch's public state)."""
        return self._side_array(self.insertions, "_arr_i"), \
            self._side_array(self.deletions, "_arr_d")

    def _side_array(self, x, slot: str) -> np.ndarray:
        if isinstance(x, ArcArray):
            return x.a
        key = (id(x), len(x))
        cached = self.__dict__.get(slot)
        if cached is None or cached[0] != key or cached[1] is not x:
            a = np.fromiter(itertools.chain.from_iterable(x), dtype=np.int64,
                            count=2 * len(x)).reshape(-1, 2)
            cached = (key, x, a)
            self.__dict__[slot] = cached
        return cached[2]

    def _keys(self):
        """u << 32 | v keys when every id fits 31 bits, else None."""
        try:
            i, d = self.arrays()
        except OverflowError:
            return None
        for a in (i, d):
            if a.size and (a.min() < 0 or a.max() > MAX_NODE_ID):
                return None
        return (i[:, 0] << 32) | i[:, 1], (d[:, 0] << 32) | d[:, 1]

    def _sorted_keys(self):
        """(sorted insertion keys, sorted deletion keys), or None when an id
        does not fit 31 bits; cached while the batch's arrays are the same
        objects (validate_shape and is_symmetric share one sort)."""
        try:
            i, d = self.arrays()
        except OverflowError:
            return None
        c = self.__dict__.get("_skeys")
        if c is not None and c[0] is i and c[1] is d:
            return c[2]
        k = self._keys()
        out = None if k is None else (np.sort(k[0]), np.sort(k[1]))
        self.__dict__["_skeys"] = (i, d, out)
        return out

    def validate_shape(self) -> None:
        """Duplicates and overlap (graph.py:46-59)."""
        sk = self._sorted_keys()
        if sk is not None:          # vectorised test; messages from the exact path
            ki, kd = sk
            if not ((ki[1:] == ki[:-1]).any() or (kd[1:] == kd[:-1]).any() or
                    (ki.size and kd.size and
                     np.intersect1d(ki, kd, assume_unique=True).size)):
                return
        ins, dels = set(self.insertions), set(self.deletions)
        if len(ins) != len(self.insertions):
            raise BatchPreconditionError(
                f"duplicate insertion of arc {_first_duplicate(self.insertions)}")
        if len(dels) != len(self.deletions):
            raise BatchPreconditionError(
                f"duplicate deletion of arc {_first_duplicate(self.deletions)}")
        overlap = ins & dels
        if overlap:
            raise BatchPreconditionError(
                f"arc {min(overlap)} appears in both insertions and deletions")

    def is_symmetric(self) -> bool:
        """Both lists closed under reversal (graph.py:61-65)."""
        sk = self._sorted_keys()
        if sk is not None:
            # reversal is a bijection, so "closed under it" = equal key sets
            return all(np.array_equal(_unique_of_sorted(a),
                                      sorted_unique(((a & 0xFFFFFFFF) << 32) | (a >> 32)))
                       for a in sk)
        ins, dels = set(self.insertions), set(self.deletions)
        return all((v, u) in ins for u, v in ins) and \
            all((v, u) in dels for u, v in dels)

    def __len__(self) -> int:
        return len(self.insertions) + len(self.deletions)


def _first_duplicate(arcs: Sequence[Arc]) -> Arc:
    seen = set()
    for a in arcs:
        if a in seen:
            return a
        seen.add(a)
    return arcs[0]


def sorted_unique(a: np.ndarray) -> np.ndarray:
    """np.unique for int64 keys as sort + run mask (same result, much faster
    than numpy 2.3's np.unique on large arrays)."""
    return _unique_of_sorted(np.sort(np.asarray(a, dtype=np.int64)))


def _unique_of_sorted(a: np.ndarray) -> np.ndarray:
    if a.size > 1:
        keep = np.empty(a.size, dtype=bool)
        keep[0] = True
        np.not_equal(a[1:], a[:-1], out=keep[1:])
        a = a[keep]
    return a


class Graph:
    """Mutable directed graph over the fixed universe 0..node_count-1."""

    def __init__(self, node_count: int):
        if node_count < 0:
            raise NodeRangeError(f"node_count must be >= 0, got {node_count}")
        self._n = int(node_count)
        self._keys = np.empty(0, dtype=np.int64)   # sorted unique u*n+v
        self._version = 0
        self._cache: dict = {}
        self._device = None    # (version, DeviceGraph) set by the engine

    # ---- construction
    @classmethod
    def from_edges(cls, node_count: int, edges, undirected: bool = False) -> "Graph":
        """graph.py:101-116: duplicates collapse; undirected adds reversals."""
        g = cls(node_count)
        e = np.asarray(edges if isinstance(edges, np.ndarray) else list(edges),
                       dtype=np.int64).reshape(-1, 2)
        if e.size:
            bad = (e < 0) | (e >= g._n)
            if bad.any():
                v = int(e[bad][0])
                raise NodeRangeError(f"node id {v} outside universe [0, {g._n})")
        src, dst = e[:, 0], e[:, 1]
        if undirected:
            src, dst = np.concatenate([src, dst]), np.concatenate([dst, src])
        g._keys = sorted_unique(src * g._n + dst)
        g._version += 1
        return g

    @classmethod
    def from_csr(cls, node_count: int, indptr, indices) -> "Graph":
        """Adopt a canonical CSR (rows sorted ascending, no duplicates)."""
        g = cls(node_count)
        indptr = np.asarray(indptr, dtype=np.int64)
        indices = np.asarray(indices, dtype=np.int32)
        rows = np.repeat(np.arange(node_count, dtype=np.int64), np.diff(indptr))
        g._keys = rows * g._n + indices
        g._cache["csr"] = (g._version + 1, indptr, indices)
        g._version += 1
        return g

    # ---- read access
    @property
    def node_count(self) -> int:
        return self._n

    @property
    def arc_count(self) -> int:
        return int(self._keys.size)

    @property
    def version(self) -> int:
        """Monotone counter bumped by every mutating call (graph.py:128-131)."""
        return self._version

    def _check_node(self, v: int) -> None:
        if not 0 <= v < self._n:
            raise NodeRangeError(f"node id {v} outside universe [0, {self._n})")

    def has_arc(self, u: int, v: int) -> bool:
        self._check_node(u)
        self._check_node(v)
        k = u * self._n + v
        i = np.searchsorted(self._keys, k)
        return bool(i < self._keys.size and self._keys[i] == k)

    def _has_keys(self, keys: np.ndarray) -> np.ndarray:
        if not keys.size or not self._keys.size:
            return np.zeros(keys.size, dtype=bool)
        i = np.searchsorted(self._keys, keys)
        i = np.minimum(i, self._keys.size - 1)
        return self._keys[i] == keys

    def csr_arrays(self) -> tuple[np.ndarray, np.ndarray]:
        """(indptr int64[n+1], indices int32[nnz]), rows ascending."""
        c = self._cache.get("csr")
        if c is None or c[0] != self._version:
            rows = self._keys // self._n if self._n else self._keys
            indptr = np.zeros(self._n + 1, dtype=np.int64)
            if self._n:
                np.cumsum(np.bincount(rows, minlength=self._n), out=indptr[1:])
            indices = (self._keys - rows * self._n).astype(np.int32)
            c = (self._version, indptr, indices)
            self._cache["csr"] = c
        return c[1], c[2]

    def _in_csr(self):
        c = self._cache.get("in")
        if c is None or c[0] != self._version:
            n = self._n
            rows = self._keys // n if n else self._keys
            cols = self._keys - rows * n
            tk = np.sort(cols * n + rows)
            indptr = np.zeros(n + 1, dtype=np.int64)
            if n:
                np.cumsum(np.bincount(cols, minlength=n), out=indptr[1:])
            c = (self._version, indptr, (tk - (tk // n) * n).astype(np.int64) if n else tk)
            self._cache["in"] = c
        return c[1], c[2]

    def out_neighbors(self, v: int) -> Iterator[int]:
        self._check_node(v)
        ip, ix = self.csr_arrays()
        return iter(ix[ip[v]:ip[v + 1]].tolist())

    def in_neighbors(self, v: int) -> Iterator[int]:
        self._check_node(v)
        ip, ix = self._in_csr()
        return iter(ix[ip[v]:ip[v + 1]].tolist())

    def out_degree(self, v: int) -> int:
        self._check_node(v)
        ip, _ = self.csr_arrays()
        return int(ip[v + 1] - ip[v])

    def in_degree(self, v: int) -> int:
        self._check_node(v)
        ip, _ = self._in_csr()
        return int(ip[v + 1] - ip[v])

    def out_degrees(self) -> np.ndarray:
        ip, _ = self.csr_arrays()
        return np.diff(ip)

    def max_out_degree(self) -> int:
        """graph.py:154-158 (cached per version: init asks twice)."""
        c = self._cache.get("maxdeg")
        if c is None or c[0] != self._version:
            c = (self._version, int(self.out_degrees().max()) if self._n else 0)
            self._cache["maxdeg"] = c
        return c[1]

    def arcs(self) -> Iterator[Arc]:
        n = self._n
        for k in self._keys.tolist():
            yield (k // n, k % n)

    def is_symmetric(self) -> bool:
        """Arc set closed under reversal (graph.py:168-175)."""
        c = self._cache.get("sym")
        if c is None or c[0] != self._version:
            n = self._n
            rows = self._keys // n if n else self._keys
            rev = np.sort((self._keys - rows * n) * n + rows) if n else self._keys
            c = (self._version, bool(np.array_equal(rev, self._keys)))
            self._cache["sym"] = c
        return c[1]

    def out_csr(self):
        """scipy view of the canonical CSR (graph.py:177-197), for callers
        that expect the reference's return type."""
        c = self._cache.get("scipy_csr")
        if c is None or c[0] != self._version:   # cached per version (graph.py:184)
            from scipy import sparse
            ip, ix = self.csr_arrays()
            c = (self._version,
                 sparse.csr_matrix((np.ones(ix.size), ix, ip), shape=(self._n, self._n)))
            self._cache["scipy_csr"] = c
        return c[1]

    # ---- mutation
    def apply_batch(self, batch: EdgeBatch) -> None:
        self.validate_batch(batch)
        self.remove_arcs(batch.deletions, _validated=True)
        self.insert_arcs(batch.insertions, _validated=True)

    def validate_batch(self, batch: EdgeBatch) -> None:
        """graph.py:207-220."""
        batch.validate_shape()
        n = self._n
        check_batch_arcs(batch, n, self._check_node,
                         lambda a: self._has_keys(a[:, 0] * n + a[:, 1]))

    def _arc_keys(self, arcs) -> np.ndarray:
        if isinstance(arcs, ArcArray):
            return arcs.a[:, 0] * self._n + arcs.a[:, 1]
        return np.array([u * self._n + v for u, v in arcs], dtype=np.int64)

    def insert_arcs(self, arcs: Sequence[Arc], _validated: bool = False) -> None:
        if not _validated:
            self.validate_batch(EdgeBatch(insertions=_arcs_in(arcs)))
        if len(arcs):
            k = np.sort(self._arc_keys(arcs))
            self._keys = np.insert(self._keys, np.searchsorted(self._keys, k), k)
        self._version += 1

    def remove_arcs(self, arcs: Sequence[Arc], _validated: bool = False) -> None:
        if not _validated:
            self.validate_batch(EdgeBatch(deletions=_arcs_in(arcs)))
        if len(arcs):
            k = self._arc_keys(arcs)
            self._keys = np.delete(self._keys, np.searchsorted(self._keys, k))
        self._version += 1

    def __repr__(self) -> str:
        return f"Graph(nodes={self._n}, arcs={self.arc_count})"


def csr_of(g) -> tuple[np.ndarray, np.ndarray]:
    """Canonical CSR arrays of any graph exposing the reference surface."""
    if hasattr(g, "csr_arrays"):
        return g.csr_arrays()
    A = g.out_csr()
    if hasattr(A, "has_sorted_indices") and not A.has_sorted_indices:
        A = A.sorted_indices()
    return (np.ascontiguousarray(A.indptr, dtype=np.int64),
            np.ascontiguousarray(A.indices, dtype=np.int32))
