"""Steady-state phase trace of one C5 update (KB_TRACE around that call
only): a warm-up update on a throwaway copy first, as bench.py does."""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1807_03847_b200 as P  # noqa: E402
from paper_1807_03847_b200 import generators as G  # noqa: E402

n = 1 << int(os.environ.get("SCALE", "24"))
crit = P.Criterion.top_k(100, 1e-6)


def batch_for(g, b, seed):
    deg = g.out_degrees()
    rng = np.random.default_rng(seed)
    e = rng.integers(0, n, size=(3 * b, 2))
    e = e[e[:, 0] != e[:, 1]]
    e = np.unique(np.sort(e, axis=1), axis=0)
    e = e[(deg[e[:, 0]] + 1 < deg.max()) & (deg[e[:, 1]] + 1 < deg.max())][:b]
    e = e[~g._present(e)]
    return P.EdgeBatch(insertions=np.concatenate([e, e[:, ::-1]]))


gw = G.rmat_graph(n, edge_factor=16, seed=42)
sw = P.init(gw, crit, undirected=True, max_iterations=200)
P.run(sw, gw)
P.update_batch(sw, gw, batch_for(gw, 2000, 1234))
del sw, gw
gc.collect()
g = G.rmat_graph(n, edge_factor=16, seed=42)
st = P.init(g, crit, undirected=True, max_iterations=200)
P.run(st, g)
for b in [int(x) for x in os.environ.get("EDGES", "100,10000,100000").split(",")]:
    batch = batch_for(g, b, 7 + b)
    t0 = time.perf_counter()
    P.update_batch(st, g, batch)
    t_plain = time.perf_counter() - t0
    batch = batch_for(g, b, 8 + b)
    os.environ["KB_TRACE"] = "1"
    t0 = time.perf_counter()
    P.update_batch(st, g, batch)
    t_tr = time.perf_counter() - t0
    del os.environ["KB_TRACE"]
    s = st.last_update_stats
    print(f"batch {b}: plain {t_plain*1e3:.2f} ms, traced {t_tr*1e3:.2f} ms, "
          f"levels {s.level_sizes} abort {s.aborted_level}", flush=True)
    t0 = time.perf_counter()
    P.run(P.init(g, crit, undirected=True, max_iterations=200), g)
    print(f"  static recompute {1e3*(time.perf_counter()-t0):.2f} ms", flush=True)
