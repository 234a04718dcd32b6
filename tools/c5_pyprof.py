"""Python-side profile of steady-state C5 updates (cProfile around
update_batch), to split host work from the device phases KB_TRACE shows."""
import cProfile
import gc
import os
import pstats
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


g = G.rmat_graph(n, edge_factor=16, seed=42)
st = P.init(g, crit, undirected=True, max_iterations=200)
P.run(st, g)
P.update_batch(st, g, batch_for(g, 2000, 1234))
for b in [int(x) for x in os.environ.get("EDGES", "10000,100000").split(",")]:
    for rep in range(3):
        batch = batch_for(g, b, 7 + b + rep)
        pr = cProfile.Profile()
        t0 = time.perf_counter()
        pr.enable()
        P.update_batch(st, g, batch)
        pr.disable()
        t = time.perf_counter() - t0
        s = st.last_update_stats
        print(f"batch {b} rep {rep}: {t*1e3:.2f} ms levels {s.level_sizes} abort {s.aborted_level}",
              flush=True)
    pstats.Stats(pr).sort_stats("tottime").print_stats(14)
