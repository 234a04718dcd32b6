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
from .errors import ParameterError


class DeviceResidentGraph:
    """node_count / version / max_out_degree() / is_symmetric() / out_csr()
    over a device graph (graph.py:80-255 surface, read-only)."""

    def __init__(self, dg: DeviceGraph):
        self._dg = dg
        info = dg.info()
        self.node_count = int(info.n)
        self.arc_count = int(info.nnz)
        self._max = int(info.max_out_degree)
        self.version = 1
        self._device = (self.version, dg)
        self._csr = None

    @property
    def device_graph(self) -> DeviceGraph:
        return self._dg

    def max_out_degree(self) -> int:
        return self._max

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

    def out_degrees(self) -> np.ndarray:
        return np.diff(self.csr_arrays()[0])

    def out_csr(self):
        from scipy import sparse
        ip, ix = self.csr_arrays()
        return sparse.csr_matrix((np.ones(ix.size), ix, ip),
                                 shape=(self.node_count, self.node_count))


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
