"""Host-side phases of update_batch for the C5 1e5-edge batch on C2."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1807_03847_b200 as P
from paper_1807_03847_b200 import generators as G

n = 1 << int(os.environ.get("SCALE", "24"))
b = int(os.environ.get("EDGES", "100000"))
g = G.rmat_graph(n, edge_factor=16, seed=42)
crit = P.Criterion.top_k(100, 1e-6)
st = P.init(g, crit, undirected=True, max_iterations=200)
P.run(st, g)
deg = g.out_degrees()
rng = np.random.default_rng(7)
e = rng.integers(0, n, size=(3 * b, 2))
e = e[e[:, 0] != e[:, 1]]
e = np.unique(np.sort(e, axis=1), axis=0)
e = e[(deg[e[:, 0]] + 1 < deg.max()) & (deg[e[:, 1]] + 1 < deg.max())][:b]
e = e[~g._present(e)]
arcs = np.concatenate([e, e[:, ::-1]])
t = [time.perf_counter()]
batch = P.EdgeBatch(insertions=arcs); t.append(time.perf_counter())
batch.arrays(); t.append(time.perf_counter())
g.validate_batch(batch); t.append(time.perf_counter())
batch.is_symmetric(); t.append(time.perf_counter())
g.max_degree_after(batch); t.append(time.perf_counter())
P.update_batch(st, g, batch); t.append(time.perf_counter())
names = ["EdgeBatch", "arrays", "validate_batch", "is_symmetric", "max_degree_after", "update_batch(all)"]
print({k: round((t[i + 1] - t[i]) * 1e3, 2) for i, k in enumerate(names)})
