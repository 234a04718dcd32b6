"""Device-side instance generators (katzbounds.generate, generate.py:38-103).

``rmat_graph``/``grid_graph`` build the graph directly in HBM with kernels
that replay the reference generator bit for bit (kb_graph_create_rmat /
kb_graph_create_grid) and return a ``DeviceResidentGraph``: a graph object
with the reference's duck-typed surface whose arcs live only on the device
(the host CSR is downloaded on demand).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .engine import DeviceGraph
from .errors import NodeRangeError, ParameterError
from .graph import EdgeBatch, check_batch_arcs


class DeviceResidentGraph:
    """A graph whose arcs live only in HBM, with the reference's Graph surface
    (graph.py:80-255): node_count, arc_count, version, has_arc, out_degrees,
    max_out_degree, is_symmetric, out_csr, in_neighbors, validate_batch,
    insert_arcs, remove_arcs, apply_batch.  Mutations edit the device
    CSR-with-slack in place; nothing is mirrored on the host."""

    def __init__(self, dg: DeviceGraph):
        self._dg = dg
        info = dg.info()
        self.node_count = int(info.n)
        self._version = 1
        self._device = (self._version, dg)
        self._csr = None

    @property
    def version(self) -> int:
        return self._version

    def _bump(self):
        self._version += 1
        self._device = (self._version, self._dg)
        self._csr = None

    @property
    def device_graph(self) -> DeviceGraph:
        return self._dg

    @property
    def arc_count(self) -> int:
        return int(self._dg.info().nnz)

    def _check_node(self, v: int) -> None:
        if not 0 <= v < self.node_count:
            raise NodeRangeError(f"node id {v} outside universe [0, {self.node_count})")

    def _arcs(self, arcs) -> np.ndarray:
        a = np.ascontiguousarray(np.asarray(arcs, dtype=np.int64).reshape(-1, 2))
        if a.size and (a.min() < 0 or a.max() >= self.node_count):
            bad = (a < 0) | (a >= self.node_count)
            if bad.any():
                self._check_node(int(a[bad][0]))
        return a

    def _present(self, a: np.ndarray) -> np.ndarray:
        out = np.zeros(a.shape[0], dtype=np.uint8)
        if a.shape[0]:
            _lib.check(_lib.lib().kb_graph_has_arcs(self._dg.handle, _lib.ptr(a), a.shape[0],
                                                    _lib.ptr(out)))
        return out.astype(bool)

    def has_arc(self, u: int, v: int) -> bool:
        self._check_node(u)
        self._check_node(v)
        return bool(self._present(self._arcs([(u, v)]))[0])

    def max_out_degree(self) -> int:
        c = getattr(self, "_maxdeg", None)
        if c is None or c[0] != self.version:        # cached per version
            c = (self.version, self.max_degree_after(EdgeBatch()))
            self._maxdeg = c
        return c[1]

    def max_degree_after(self, batch: EdgeBatch) -> int:
        """dynamic.py:151-157 evaluated on the device."""
        i, d = (self._arcs(a) for a in batch.arrays())
        out = ctypes.c_int64()
        _lib.check(_lib.lib().kb_graph_max_degree_after(self._dg.handle, _lib.ptr(i), i.shape[0],
                                                        _lib.ptr(d), d.shape[0],
                                                        ctypes.byref(out)))
        return int(out.value)

    def out_degrees(self) -> np.ndarray:
        out = np.empty(self.node_count, dtype=np.int64)
        _lib.check(_lib.lib().kb_graph_out_degrees(self._dg.handle, _lib.ptr(out)))
        return out

    def is_symmetric(self) -> bool:
        return self._dg.is_symmetric()

    def csr_arrays(self):
        if self._csr is None:
            indptr = np.empty(self.node_count + 1, dtype=np.int64)
            indices = np.empty(self.arc_count, dtype=np.int32)
            _lib.check(_lib.lib().kb_graph_get_csr(self._dg.handle, _lib.ptr(indptr),
                                                   _lib.ptr(indices)))
            self._csr = (indptr, indices)
        return self._csr

    def out_neighbors(self, v: int):
        self._check_node(v)
        ip, ix = self.csr_arrays()
        return iter(ix[ip[v]:ip[v + 1]].tolist())

    def in_neighbors(self, v: int):
        self._check_node(v)
        ip, ix = self.csr_arrays()
        rows = np.repeat(np.arange(self.node_count), np.diff(ip))
        return iter(rows[ix == v].tolist())

    def arcs(self):
        ip, ix = self.csr_arrays()
        for u in range(self.node_count):
            for v in ix[ip[u]:ip[u + 1]].tolist():
                yield (u, v)

    def out_csr(self):
        c = getattr(self, "_scipy", None)
        if c is None or c[0] != self.version:     # cached per version (graph.py:184)
            from scipy import sparse
            ip, ix = self.csr_arrays()
            c = (self.version, sparse.csr_matrix((np.ones(ix.size), ix, ip),
                                                 shape=(self.node_count, self.node_count)))
            self._scipy = c
        return c[1]

    # ---- mutation (graph.py:201-237)
    def validate_batch(self, batch: EdgeBatch) -> None:
        """graph.py:207-220 (presence tested on the device)."""
        batch.validate_shape()
        check_batch_arcs(batch, self.node_count, self._check_node, self._present)

    def _apply(self, ins, dels):
        i, d = self._arcs(ins), self._arcs(dels)
        _lib.check(_lib.lib().kb_graph_apply_batch(self._dg.handle, _lib.ptr(i), i.shape[0],
                                                   _lib.ptr(d), d.shape[0]))

    def apply_batch(self, batch: EdgeBatch) -> None:
        self.validate_batch(batch)
        self.remove_arcs(batch.deletions, _validated=True)
        self.insert_arcs(batch.insertions, _validated=True)

    def insert_arcs(self, arcs, _validated: bool = False) -> None:
        if not _validated:
            self.validate_batch(EdgeBatch(insertions=list(arcs)))
        self._apply(arcs, [])
        self._bump()

    def remove_arcs(self, arcs, _validated: bool = False) -> None:
        if not _validated:
            self.validate_batch(EdgeBatch(deletions=list(arcs)))
        self._apply([], arcs)
        self._bump()

    def _note_device_update(self) -> None:
        """update_batch already edited the device arcs: deletions then
        insertions, two version bumps (dynamic.py:170, :199)."""
        self._bump()
        self._bump()


def _wrap(h, device) -> DeviceGraph:
    dg = DeviceGraph.__new__(DeviceGraph)
    dg._h = h
    dg.device = device
    dg._L = _lib.lib()
    return dg


def pcg64_state(seed: int) -> np.ndarray:
    """{state_hi, state_lo, inc_hi, inc_lo} of np.random.default_rng(seed)
    (generate.py:68) -- the seeding runs numpy's SeedSequence on the host."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    M = (1 << 64) - 1
    return np.array([s >> 64, s & M, inc >> 64, inc & M], dtype=np.uint64)


def rmat_graph(n: int, edge_factor: int = 8, seed: int = 0, *, device: int = 0,
               quadrants=(0.57, 0.19, 0.19, 0.05), split_threshold: int = 0,
               hot_size: int = -1) -> DeviceResidentGraph:
    """generate('rmat', n, seed=seed, edge_factor=edge_factor) loaded with
    undirected=True, built on the device."""
    if not (n >= 2 and (n & (n - 1)) == 0):
        raise ParameterError(f"rmat model needs a power-of-two node count >= 2, got {n}")
    if edge_factor < 1:
        raise ParameterError(f"edge_factor must be >= 1, got {edge_factor}")
    a, b, c, _ = quadrants
    if abs(sum(quadrants) - 1.0) >= 1e-9:
        raise ParameterError("quadrant probabilities must sum to 1")
    ab = a + b          # the same Python float expressions as generate.py:73-74
    abc = a + b + c
    state = pcg64_state(seed)
    h = ctypes.c_void_p()
    _lib.check(_lib.lib().kb_graph_create_rmat(device, n.bit_length() - 1, edge_factor,
                                               _lib.ptr(state), a, ab, abc, split_threshold,
                                               hot_size, ctypes.byref(h)))
    return DeviceResidentGraph(_wrap(h, device))


def grid_graph(n: int, *, device: int = 0, split_threshold: int = 0,
               hot_size: int = -1) -> DeviceResidentGraph:
    """generate('grid', n) loaded with undirected=True, built on the device."""
    if n < 1:
        raise ParameterError(f"grid model needs >= 1 node, got {n}")
    h = ctypes.c_void_p()
    _lib.check(_lib.lib().kb_graph_create_grid(device, n, split_threshold, hot_size,
                                               ctypes.byref(h)))
    return DeviceResidentGraph(_wrap(h, device))


MODELS = ("complete", "star", "path", "grid", "rmat")


def _need(cond: bool, message: str) -> None:
    if not cond:
        raise ParameterError(message)


def _upper_pairs(g: DeviceResidentGraph) -> np.ndarray:
    """(u, v) with u < v of a symmetric device graph, in (u, v) order."""
    ip, ix = g.csr_arrays()
    rows = np.repeat(np.arange(g.node_count, dtype=np.int64), np.diff(ip))
    keep = rows < ix
    return np.stack([rows[keep], ix[keep].astype(np.int64)], axis=1)


def generate(model: str, n: int, *, seed: int = 0, edge_factor: int = 8,
             as_array: bool = False, device: int = 0):
    """generate.py:89-103: the undirected edge pairs (u < v) of a benchmark
    instance, in the reference's order.  rmat and grid come from the device
    generators (bit-identical replays); as_array=True returns an (m, 2)
    int64 array instead of a list of tuples."""
    if model == "complete":
        _need(n >= 1, f"complete model needs >= 1 node, got {n}")
        iu = np.triu_indices(n, 1)
        e = np.stack([iu[0], iu[1]], axis=1).astype(np.int64)
    elif model == "star":
        _need(n >= 1, f"star model needs >= 1 node, got {n}")
        e = np.stack([np.zeros(n - 1, dtype=np.int64), np.arange(1, n, dtype=np.int64)], axis=1)
    elif model == "path":
        _need(n >= 1, f"path model needs >= 1 node, got {n}")
        a = np.arange(n - 1, dtype=np.int64)
        e = np.stack([a, a + 1], axis=1)
    elif model == "grid":
        _need(n >= 1, f"grid model needs >= 1 node, got {n}")
        e = _upper_pairs(grid_graph(n, device=device)) if n > 1 else np.zeros((0, 2), np.int64)
    elif model == "rmat":
        _need(n >= 2 and (n & (n - 1)) == 0,
              f"rmat model needs a power-of-two node count >= 2, got {n}")
        _need(edge_factor >= 1, f"edge_factor must be >= 1, got {edge_factor}")
        e = _upper_pairs(rmat_graph(n, edge_factor=edge_factor, seed=seed, device=device))
    else:
        raise ParameterError(f"unknown model {model!r}; choose one of {', '.join(MODELS)}")
    e = e.reshape(-1, 2)
    if as_array:
        return e
    return list(zip(e[:, 0].tolist(), e[:, 1].tolist()))
