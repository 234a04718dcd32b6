"""Sweep K1 tuning knobs on the C2 graph; prints ms/iteration per variant and
checks every variant produces bit-identical katz vectors."""
from __future__ import annotations

import ctypes
import hashlib
import itertools
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1807_03847_b200 as P  # noqa: E402
from paper_1807_03847_b200 import _lib  # noqa: E402
from paper_1807_03847_b200 import generators as G  # noqa: E402


def main():
    scale = int(os.environ.get("SCALE", "24"))
    iters = int(os.environ.get("ITERS", "7"))
    grid = json.loads(os.environ.get("GRID", '{"k1.depth":[1,2,3],"k1.hot":[0,12288,24576],"k1.xload":[0,1,2]}'))
    L = _lib.lib()
    splits = json.loads(os.environ.get("SPLITS", "[8192]"))
    crit = P.Criterion.top_k(100, 1e-6)
    keys = list(grid)
    ref = None
    for split, vals in itertools.product(splits, itertools.product(*[grid[k] for k in keys])):
        if split != getattr(main, "_split", None):
            t0 = time.time()
            g = G.rmat_graph(1 << scale, edge_factor=16, seed=42, split_threshold=split)
            main._split = split
            inf = g.device_graph.info()
            print(f"s{scale} split={split}: heavy_rows={inf.heavy_rows} segments={inf.segments} "
                  f"slices={inf.slices} elems={inf.sell_elems} ({time.time()-t0:.2f}s)", flush=True)
        for k, v in zip(keys, vals):
            L.kb_tune(k.encode(), int(v))
        st = P.init(g, crit, undirected=True)
        P.iterate_once(st, g)  # warm: first iteration also writes empty rows
        for _ in range(iters - 1):
            P.iterate_once(st, g)
        info = st._info()
        katz = st.katz
        h = hashlib.sha256(katz.tobytes()).hexdigest()[:16]
        if ref is None:
            ref = h
        ms = info.spmv_ms / max(1, info.spmv_launches)
        print(json.dumps({"split": split, "cfg": dict(zip(keys, vals)), "k1_ms": round(ms, 4),
                          "katz": h, "same": h == ref}), flush=True)
        del st


if __name__ == "__main__":
    main()
