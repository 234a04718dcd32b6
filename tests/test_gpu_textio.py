"""Device text ingestion (kb_text_scan + kb_graph_create_text) against the
reference's own outcomes (tests/golden/textio.json from
make_textio_golden.py): the same graphs, and for bad inputs the same error
class, message and line number (graph.py:260-342, dynamic.py:216-253)."""
from __future__ import annotations

import io
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_1807_03847_b200")
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def tio():
    with open(os.path.join(GOLDEN, "textio.json")) as fh:
        return json.load(fh)


def outcome(fn):
    try:
        return {"ok": fn()}
    except P.KatzError as e:
        return {"error": type(e).__name__, "message": str(e), "line": getattr(e, "line", None)}
    except UnicodeDecodeError as e:
        return {"error": "UnicodeDecodeError", "message": str(e), "line": None}


def summary(g):
    return {"n": g.node_count, "arcs": [list(a) for a in sorted(g.arcs())]}


def test_edge_lists_match_reference(tio, tmp_path):
    for i, rec in enumerate(tio["edges"]):
        data = bytes.fromhex(rec["hex"])
        path = tmp_path / f"e{i}.txt"
        path.write_bytes(data)
        for und in (0, 1):
            got = outcome(lambda: summary(P.load_edge_list(str(path), undirected=bool(und))))
            assert got == rec[f"path_{und}"], (data, und)
        assert outcome(lambda: summary(P.load_edge_list(io.BytesIO(data)))) == rec["bytesio"], data


def test_batch_files_match_reference(tio, tmp_path):
    def summ(bs):
        return [{"ins": [list(a) for a in b.insertions],
                 "dels": [list(a) for a in b.deletions]} for b in bs]
    for i, rec in enumerate(tio["batches"]):
        data = bytes.fromhex(rec["hex"])
        path = tmp_path / f"b{i}.txt"
        path.write_bytes(data)
        assert outcome(lambda: summ(P.load_batches(str(path)))) == rec["path"], data
        if "stringio" in rec:
            text = data.decode("utf-8")
            assert outcome(lambda: summ(P.load_batches(io.StringIO(text)))) == rec["stringio"]


def _snap_like() -> bytes:
    rng = np.random.default_rng(3)
    lines = ["# Directed graph (each unordered pair of nodes is saved once)",
             "# Nodes: 5000 Edges: 40000", "# FromNodeId\tToNodeId"]
    for _ in range(40000):
        u, v = rng.integers(0, 5000, size=2)
        sep = "\t" if rng.random() < 0.5 else " "
        end = "\r" if rng.random() < 0.1 else ""
        lines.append(f"{u}{sep}{v}{end}")
        if rng.random() < 0.01:
            lines.append("% interleaved comment")
    return ("\n".join(lines) + "\n").encode()


def test_snap_like_file_and_engine_reuse(tio, tmp_path):
    path = tmp_path / "snap.txt"
    path.write_bytes(_snap_like())
    g = P.load_edge_list(str(path), undirected=True)
    ref = tio["snap_like"]
    ip, ix = g.csr_arrays()
    assert g.node_count == ref["n"] and int(ip[-1]) == ref["nnz"]
    assert int(ip.sum()) == ref["indptr_sum"] and int(ix.astype(np.int64).sum()) == ref["indices_sum"]
    # the loaded graph carries its device copy: the engine runs without re-upload
    dg = g._device[1]
    res = P.run(P.init(g, P.Criterion.top_k(10, 1e-8), undirected=True), g)
    assert g._device[1] is dg
    g2 = P.Graph.from_csr(g.node_count, ip, ix)
    res2 = P.run(P.init(g2, P.Criterion.top_k(10, 1e-8), undirected=True), g2)
    np.testing.assert_array_equal(res.order, res2.order)
    r = P.load_edge_list(str(path), undirected=True, resident=True)
    assert r.arc_count == ref["nnz"] and r.is_symmetric()


def test_large_generated_edge_list_roundtrip(tmp_path):
    """dumps_edge_list -> load_edge_list on an R-MAT s16 graph (1.8M arcs)."""
    from paper_1807_03847_b200 import generators as G
    g = G.rmat_graph(1 << 16, edge_factor=16, seed=42)
    ip, ix = g.csr_arrays()
    rows = np.repeat(np.arange(g.node_count), np.diff(ip))
    keep = rows < ix
    text = P.dumps_edge_list(g.node_count, zip(rows[keep].tolist(), ix[keep].tolist()))
    path = tmp_path / "rmat.txt"
    path.write_text(text)
    h = P.load_edge_list(str(path), undirected=True)
    ip2, ix2 = h.csr_arrays()
    np.testing.assert_array_equal(ip2, ip)
    np.testing.assert_array_equal(ix2, ix)


def test_generate_matches_reference_digests(tio):
    import hashlib
    for rec in tio["generate"]:
        e = P.generate(rec["model"], rec["n"], as_array=True, **rec["kw"])
        assert e.shape[0] == rec["m"], rec
        assert hashlib.sha256(np.ascontiguousarray(e, dtype=np.int64).tobytes()).hexdigest()[:16] \
            == rec["sha"], rec
    assert P.generate("star", 4) == [(0, 1), (0, 2), (0, 3)]
    with pytest.raises(P.ParameterError):
        P.generate("rmat", 3)
    with pytest.raises(P.ParameterError):
        P.generate("nope", 3)
