"""Why is the first update_batch on a graph slow?  Pool reserve/used bytes
and wall time around each step of the C5 setup (KB_TRACE=1 adds phases)."""
from __future__ import annotations

import gc
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_03847_b200 as P  # noqa: E402
from paper_1807_03847_b200 import _lib  # noqa: E402
from paper_1807_03847_b200 import generators as G  # noqa: E402

L = _lib.lib()


def pool(tag, t0):
    info = np.zeros(4, dtype=np.int64)
    _lib.check(L.kb_pool_info(0, _lib.ptr(info)))
    print(f"{tag:28s} {time.perf_counter() - t0:8.3f}s reserved {info[0] / 2**30:7.2f} GiB "
          f"(high {info[1] / 2**30:7.2f}) used {info[2] / 2**30:7.2f} GiB (high {info[3] / 2**30:7.2f})",
          flush=True)


def batch_for(g, n, k, seed):
    deg = g.out_degrees()
    rw = np.random.default_rng(seed)
    c = rw.integers(0, n, size=(4 * k, 2))
    c = c[(c[:, 0] != c[:, 1]) & (deg[c[:, 0]] < 8) & (deg[c[:, 1]] < 8)]
    c = np.unique(np.sort(c, axis=1), axis=0)[:k]
    c = c[~g._present(c)]
    a = np.concatenate([c, c[:, ::-1]])
    return P.EdgeBatch(insertions=[tuple(x) for x in a.tolist()])


def main():
    n = 1 << int(os.environ.get("SCALE", "24"))
    reserve = int(float(os.environ.get("RESERVE_GB", "0")) * 2**30)
    crit = P.Criterion.top_k(100, 1e-6)
    t0 = time.perf_counter()
    pool("start", t0)
    if reserve:
        _lib.check(L.kb_pool_reserve(0, reserve))
        pool("reserved", t0)
    for rep in range(2):
        g = G.rmat_graph(n, edge_factor=16, seed=42)
        pool(f"[{rep}] graph", t0)
        st = P.init(g, crit, undirected=True, max_iterations=200)
        P.run(st, g)
        pool(f"[{rep}] run", t0)
        for k in (100, 1000):
            b = batch_for(g, n, k, 7 + k)
            t = time.perf_counter()
            P.update_batch(st, g, b)
            print(f"   update {k}: {1e3 * (time.perf_counter() - t):.1f} ms")
            pool(f"[{rep}] after update {k}", t0)
        t = time.perf_counter()
        P.run(P.init(g, crit, undirected=True, max_iterations=200), g)
        print(f"   static: {1e3 * (time.perf_counter() - t):.1f} ms")
        pool(f"[{rep}] static", t0)
        del st, g
        gc.collect()
        pool(f"[{rep}] freed", t0)


if __name__ == "__main__":
    main()
