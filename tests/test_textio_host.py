"""The host half of the text formats (the exact per-line rules the device
scanner defers to, paper_1807_03847_b200.textio) against the reference's own
outcomes (tests/golden/textio.json).  Every line goes through the host rules
here, so this checks them without a GPU; tests/test_gpu_textio.py checks the
device scanner plus the hand-off."""
from __future__ import annotations

import io
import json
import os

from paper_1807_03847_b200 import textio as T
from paper_1807_03847_b200.errors import KatzError, NodeRangeError

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _host_edges(data: bytes, undirected: bool):
    declared, arcs, seen, max_id = None, set(), False, -1
    lines = data.split(b"\n")
    if lines and lines[-1] == b"":
        lines.pop()
    for i, raw in enumerate(lines):
        r = T._edge_line(raw, i + 1, not seen)
        if r is None:
            continue
        seen = True
        if r[0] == "header":
            declared = r[1]
        else:
            arcs.add((r[1], r[2]))
            if undirected:
                arcs.add((r[2], r[1]))
            max_id = max(max_id, r[1], r[2])
    n = declared if declared is not None else max_id + 1
    if max_id >= n:
        raise NodeRangeError(f"node id {max_id} exceeds declared universe of {n}")
    return {"n": n, "arcs": [list(a) for a in sorted(arcs)]}


def _outcome(fn):
    try:
        return {"ok": fn()}
    except KatzError as e:
        return {"error": type(e).__name__, "message": str(e), "line": getattr(e, "line", None)}


def test_host_line_rules_match_reference():
    with open(os.path.join(GOLDEN, "textio.json")) as fh:
        tio = json.load(fh)
    for rec in tio["edges"]:
        data = bytes.fromhex(rec["hex"])
        for und in (0, 1):
            assert _outcome(lambda: _host_edges(data, bool(und))) == rec[f"path_{und}"], data
    for rec in tio["batches"]:
        if "stringio" not in rec:
            continue
        text = bytes.fromhex(rec["hex"]).decode("utf-8")
        got = _outcome(lambda: [{"ins": [list(a) for a in b.insertions],
                                 "dels": [list(a) for a in b.deletions]}
                                for b in T._batches_exact(text)])
        assert got == rec["stringio"], text


def test_dumps_edge_list():
    assert T.dumps_edge_list(3, [(0, 1), (1, 2)]) == "NODES 3\n0 1\n1 2\n"
    assert io.StringIO(T.dumps_edge_list(1, [])).read() == "NODES 1\n"
