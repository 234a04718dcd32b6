"""Golden outcomes of the reference's text formats (graph.py:260-342
load_edge_list, dynamic.py:216-253 load_batches), produced by running the
*reference* here:

    python tests/golden/make_textio_golden.py

Writes tests/golden/textio.json: for every input (as bytes, hex-encoded),
the resulting canonical arc list or the error class, message and line.
"""
from __future__ import annotations

import io
import json
import os
import sys
import tempfile

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import katzbounds as K  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

EDGE_CASES = [
    b"0 1\n1 2\n",
    b"# c\n% c\n\nNODES 10\n0 1\n",
    b"NODES 5\n",
    b"nodes 4\n0 3\n",
    b"0 1\nNODES 5\n",
    b"NODES 5 6\n",
    b"NODES x\n",
    b"0 1 2\n",
    b"0 -1\n",
    b"0 +1\n",
    b"0 1_0\n",
    b"0 2147483648\n",
    b"0 99\n",
    b"NODES 2\n0 5\n",
    b"0\t1\r\n2 3\r\n",
    b"  0   1  \n\x0c2 3\n",
    b"0 1\n\xff\n",
    "0 1\n# café\n1 2\n".encode(),
    "0 1\n".encode(),
    "٣ 1\n".encode(),
    b"0 1",
    b"",
    b"\n\n# only\n",
    b"0 0\n0 1\n",
    b"0 1\n0 1\n1 0\n",
    b"-0 1\n",
    b"00012 3\n",
    b"NODES 3\nNODES 4\n",
    b"# c\nNODES 7\n",
    b"\x00 1\n",
    b"1 2 \x1c\n",
    b"1 2\n\n\n3 4\n  # indented comment\n",
    b"NODES 3\n0 1\n2 3\n",
    b"0 1\nfoo bar\n",
    b"0 1\n1\n",
    "NODEſ 4\n0 1\n".encode(),
    b"0 1 # trailing\n",
    b"%%MatrixMarket\n3 4\n",
    b"\r\n0 1\r\n",
    b"0 1\r2 3\n",
]

BATCH_CASES = [
    b"+ 0 1\n- 1 2\n\n+ 2 3\n",
    b"",
    b"\n\n",
    b"+ 0 1\n* 2 3\n",
    b"+ 0\n",
    b"- 0 -1\n",
    b"+ 0 1\r\n\r\n+ 1 2\r\n",
    b"+ 0 99999999999\n",
    b"+ 0 +1\n",
    b"+ 1 2\n\n\n\n- 1 2\n",
    b"+ 1 2\n  \n- 2 3\n- 4 5\n+ 6 7\n",
    b"# comment\n+ 1 2\n",
    b"+ 1 2",
    b"+1 2 3\n",
    b"+ 1_0 2\n",
    "+ ٣ 2\n".encode(),
    b"+ 0 1\r- 1 2\n",
]


def outcome(fn):
    try:
        return {"ok": fn()}
    except K.KatzError as e:
        return {"error": type(e).__name__, "message": str(e),
                "line": getattr(e, "line", None)}
    except UnicodeDecodeError as e:
        return {"error": "UnicodeDecodeError", "message": str(e), "line": None}


def graph_summary(g, undirected):
    arcs = sorted(g.arcs())
    return {"n": g.node_count, "arcs": [list(a) for a in arcs]}


def main():
    out = {"edges": [], "batches": []}
    with tempfile.TemporaryDirectory() as tmp:
        for i, data in enumerate(EDGE_CASES):
            path = os.path.join(tmp, f"e{i}.txt")
            with open(path, "wb") as fh:
                fh.write(data)
            rec = {"hex": data.hex()}
            for und in (False, True):
                rec[f"path_{int(und)}"] = outcome(
                    lambda: graph_summary(K.load_edge_list(path, undirected=und), und))
            rec["bytesio"] = outcome(lambda: graph_summary(
                K.load_edge_list(io.BytesIO(data)), False))
            out["edges"].append(rec)
        for i, data in enumerate(BATCH_CASES):
            path = os.path.join(tmp, f"b{i}.txt")
            with open(path, "wb") as fh:
                fh.write(data)
            rec = {"hex": data.hex()}

            def summ(bs):
                return [{"ins": [list(a) for a in b.insertions],
                         "dels": [list(a) for a in b.deletions]} for b in bs]
            rec["path"] = outcome(lambda: summ(K.load_batches(path)))
            try:
                text = data.decode("utf-8")
                rec["stringio"] = outcome(lambda: summ(K.load_batches(io.StringIO(text))))
            except UnicodeDecodeError:
                pass
            out["batches"].append(rec)
    # a larger mixed file: SNAP-style comments, tabs, CRLF, duplicates
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
    big = ("\n".join(lines) + "\n").encode()
    g = K.load_edge_list(io.BytesIO(big), undirected=True)
    ip = g.out_csr().indptr
    out["snap_like"] = {"n": g.node_count, "nnz": int(ip[-1]),
                        "indptr_sum": int(np.asarray(ip, dtype=np.int64).sum()),
                        "indices_sum": int(np.asarray(g.out_csr().indices,
                                                      dtype=np.int64).sum())}
    # generate() (generate.py:89-103): edge-list digests
    import hashlib
    gen = []
    for model, n, kw in [("grid", 1, {}), ("grid", 2, {}), ("grid", 3, {}), ("grid", 10, {}),
                         ("grid", 17, {}), ("grid", 1000, {}), ("rmat", 2, {}),
                         ("rmat", 1024, {}), ("rmat", 4096, dict(seed=3, edge_factor=16)),
                         ("rmat", 1 << 15, dict(seed=42, edge_factor=16)),
                         ("star", 7, {}), ("path", 5, {}), ("complete", 6, {})]:
        e = np.asarray(K.generate(model, n, **kw), dtype=np.int64).reshape(-1, 2)
        gen.append(dict(model=model, n=n, kw=kw, m=int(e.shape[0]),
                        sha=hashlib.sha256(e.tobytes()).hexdigest()[:16]))
    out["generate"] = gen
    with open(os.path.join(HERE, "textio.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("edges", len(out["edges"]), "batches", len(out["batches"]))


if __name__ == "__main__":
    main()
