"""Edge-list and batch-file formats, parsed on the device
(reference graph.py:260-342 load_edge_list / dumps_edge_list and
dynamic.py:216-253 load_batches).

The file is memory-mapped and copied to HBM in one transfer; a kernel splits
and classifies every line (kb_text_scan).  Lines outside the plain ASCII
grammar -- non-ASCII bytes, signs, underscores, overflowing or negative ids,
wrong field counts, every NODES line -- come back as a short list and are
re-read here with the reference's exact rules, in file order, so accepted
inputs, error classes, messages and line numbers match the reference.  The
arcs go straight into the device CSR builder (kb_graph_create_text); the
returned graph already holds its device copy.
"""
from __future__ import annotations

import ctypes
import io
import logging
import mmap
import os
from pathlib import Path

import numpy as np

from . import _lib
from .errors import NodeRangeError, ParseError
from .graph import EdgeBatch, Graph

log = logging.getLogger(__name__)

MAX_NODE_ID = 2**31 - 1


class _Bytes:
    """The whole input as one read-only buffer (mmap for paths)."""

    def __init__(self, source, text_mode: bool):
        self._mm = None
        self._fh = None
        is_path = isinstance(source, (str, Path)) or hasattr(source, "__fspath__") or \
            (text_mode and isinstance(source, bytes))
        if is_path:
            if text_mode:
                # load_batches opens in text mode: newline translation applies
                with open(source, "r", encoding="utf-8") as fh:
                    self.data = fh.read().encode("utf-8", "surrogatepass")
                return
            self._fh = open(source, "rb")
            size = os.fstat(self._fh.fileno()).st_size
            if size:
                self._mm = mmap.mmap(self._fh.fileno(), 0, access=mmap.ACCESS_READ)
                self.data = self._mm
            else:
                self.data = b""
            return
        data = source.read()
        if isinstance(data, str):
            data = data.encode("utf-8", "surrogatepass")
        self.data = bytes(data)

    def __len__(self):
        return len(self.data)

    def ptr(self):
        if not len(self.data):
            return None
        self._view = np.frombuffer(self.data, dtype=np.uint8)
        return self._view.ctypes.data_as(ctypes.c_void_p)

    def line(self, start: int, end: int) -> bytes:
        return bytes(self.data[start:end])

    def close(self):
        self._view = None
        if self._mm is not None:
            self._mm.close()
        if self._fh is not None:
            self._fh.close()


class _Scan:
    def __init__(self, src: _Bytes, batches: bool, device: int):
        self.L = _lib.lib()
        h = ctypes.c_void_p()
        info = np.zeros(5, dtype=np.int64)
        _lib.check(self.L.kb_text_scan(device, src.ptr(), len(src), int(batches),
                                       ctypes.byref(h), _lib.ptr(info)))
        self.h = h
        self.device = device
        (self.n_lines, self.n_arcs, self.n_cand, self.first_arc_line,
         self.max_id) = (int(x) for x in info)

    def candidates(self) -> np.ndarray:
        out = np.zeros((self.n_cand, 3), dtype=np.int64)
        if self.n_cand:
            _lib.check(self.L.kb_text_candidates(self.h, _lib.ptr(out)))
        return out

    def lines(self):
        kind = np.empty(self.n_lines, dtype=np.uint8)
        u = np.empty(self.n_lines, dtype=np.int32)
        v = np.empty(self.n_lines, dtype=np.int32)
        if self.n_lines:
            _lib.check(self.L.kb_text_lines(self.h, _lib.ptr(kind), _lib.ptr(u), _lib.ptr(v)))
        return kind, u, v

    def close(self):
        if self.h:
            self.L.kb_text_destroy(self.h)
            self.h = None


# ---------------------------------------------------------------- edge lists

def _parse_id(token: str, lineno: int) -> int:
    """graph.py:316-326."""
    try:
        value = int(token)
    except ValueError:
        raise ParseError(f"not an integer: {token!r}", lineno) from None
    if value < 0:
        raise ParseError(f"negative node id {value}", lineno)
    if value > MAX_NODE_ID:
        raise NodeRangeError(f"line {lineno}: node id {value} overflows the 32-bit id type")
    return value


def _edge_line(raw: bytes, lineno: int, header_allowed: bool):
    """One line under the reference's rules (graph.py:283-306):
    None (blank/comment), ('header', n) or ('arc', u, v)."""
    try:
        line = raw.decode("utf-8")
    except UnicodeDecodeError:
        raise ParseError("not valid UTF-8 text", lineno) from None
    line = line.strip()
    if not line or line.startswith("#") or line.startswith("%"):
        return None
    parts = line.split()
    if header_allowed and parts[0].upper() == "NODES":
        if len(parts) != 2:
            raise ParseError("malformed NODES header", lineno)
        return ("header", _parse_id(parts[1], lineno))
    if len(parts) != 2:
        raise ParseError(f"expected two node ids, got {len(parts)} fields", lineno)
    return ("arc", _parse_id(parts[0], lineno), _parse_id(parts[1], lineno))


def load_edge_list(source, undirected: bool = False, *, device: int = 0,
                   resident: bool = False, split_threshold: int = 0, hot_size: int = -1):
    """Parse a whitespace-separated edge list (graph.py:260-313): optional
    leading "NODES <n>" header, '#'/'%' comments, blank lines, "u v" arcs;
    duplicates collapse; undirected adds reversals.  `source` is a path or
    an open text/binary stream.  Returns a Graph (resident=True: a
    DeviceResidentGraph, arcs kept only in HBM)."""
    src = _Bytes(source, text_mode=False)
    scan = None
    try:
        scan = _Scan(src, batches=False, device=device)
        declared = None
        extra = []
        content_seen = False
        max_id = scan.max_id
        for i, start, end in scan.candidates():
            lineno = int(i) + 1
            header_allowed = not content_seen and not (0 <= scan.first_arc_line < i)
            r = _edge_line(src.line(int(start), int(end)), lineno, header_allowed)
            if r is None:
                continue
            content_seen = True
            if r[0] == "header":
                declared = r[1]
            else:
                extra.append((r[1], r[2]))
                max_id = max(max_id, r[1], r[2])
        node_count = declared if declared is not None else max_id + 1
        if max_id >= node_count:
            raise NodeRangeError(
                f"node id {max_id} exceeds declared universe of {node_count}")
        if node_count == 0:
            return Graph(0)
        ex = np.ascontiguousarray(np.asarray(extra, dtype=np.int64).reshape(-1, 2))
        h = ctypes.c_void_p()
        _lib.check(scan.L.kb_graph_create_text(scan.h, node_count, int(undirected),
                                               _lib.ptr(ex) if ex.size else None, ex.shape[0],
                                               split_threshold, hot_size, ctypes.byref(h)))
    finally:
        if scan is not None:
            scan.close()
        src.close()
    from .generators import DeviceResidentGraph, _wrap
    dg = _wrap(h, device)
    if resident:
        g = DeviceResidentGraph(dg)
    else:
        nnz = int(dg.info().nnz)
        indptr = np.empty(node_count + 1, dtype=np.int64)
        indices = np.empty(nnz, dtype=np.int32)
        _lib.check(_lib.lib().kb_graph_get_csr(dg.handle, _lib.ptr(indptr), _lib.ptr(indices)))
        g = Graph.from_csr(node_count, indptr, indices)
        g._device = (g.version, dg)          # the engine reuses this device copy
    log.info("loaded edge list: %d lines, %d nodes, %d arcs", scan.n_lines, node_count,
             g.arc_count)
    return g


def dumps_edge_list(node_count: int, edges) -> str:
    """Edges with an explicit NODES header (graph.py:336-342)."""
    out = io.StringIO()
    out.write(f"NODES {node_count}\n")
    for u, v in edges:
        out.write(f"{u} {v}\n")
    return out.getvalue()


# ---------------------------------------------------------------- batch files

def _batches_exact(text: str) -> list[EdgeBatch]:
    """dynamic.py:216-253 line by line (the rare inputs the device grammar
    does not decide)."""
    batches: list[EdgeBatch] = []
    ins: list[tuple[int, int]] = []
    dels: list[tuple[int, int]] = []
    for lineno, line in enumerate(io.StringIO(text), start=1):
        line = line.strip()
        if not line:
            if ins or dels:
                batches.append(EdgeBatch(insertions=ins, deletions=dels))
                ins, dels = [], []
            continue
        parts = line.split()
        if len(parts) != 3 or parts[0] not in ("+", "-"):
            raise ParseError(f"expected '+ u v' or '- u v', got {line!r}", lineno)
        try:
            u, v = int(parts[1]), int(parts[2])
        except ValueError:
            raise ParseError(f"non-integer node id in {line!r}", lineno) from None
        if u < 0 or v < 0:
            raise ParseError(f"negative node id in {line!r}", lineno)
        (ins if parts[0] == "+" else dels).append((u, v))
    if ins or dels:
        batches.append(EdgeBatch(insertions=ins, deletions=dels))
    return batches


def load_batches(source, *, device: int = 0) -> list[EdgeBatch]:
    """Parse a batch file: "+ u v" / "- u v" lines, batches separated by
    blank lines, in file order; an empty file yields none."""
    src = _Bytes(source, text_mode=True)
    scan = None
    try:
        scan = _Scan(src, batches=True, device=device)
        if scan.n_cand:
            return _batches_exact(bytes(src.data).decode("utf-8", "surrogatepass"))
        kind, u, v = scan.lines()
    finally:
        if scan is not None:
            scan.close()
        src.close()
    # split at separator lines; each run of op lines is one batch
    op = kind != 0
    if not op.any():
        return []
    starts = np.flatnonzero(op & ~np.concatenate([[False], op[:-1]]))
    ends = np.flatnonzero(op & ~np.concatenate([op[1:], [False]])) + 1
    batches = []
    for s, e in zip(starts, ends):
        k = kind[s:e]
        pu, pv = u[s:e].tolist(), v[s:e].tolist()
        ins = [(a, b) for a, b, t in zip(pu, pv, k.tolist()) if t == 1]
        dels = [(a, b) for a, b, t in zip(pu, pv, k.tolist()) if t == 4]
        batches.append(EdgeBatch(insertions=ins, deletions=dels))
    return batches


__all__ = ["load_edge_list", "dumps_edge_list", "load_batches", "MAX_NODE_ID"]
