"""C5 correctness probe: after each batch, compare the dynamic state's top-k
with two independent static recomputes (and the static runs with each other)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1807_03847_b200 as P
from paper_1807_03847_b200 import generators as G
n = 1 << int(os.environ.get("SCALE", "24"))
crit = P.Criterion.top_k(100, 1e-6)
g = G.rmat_graph(n, edge_factor=16, seed=42)
st = P.init(g, crit, undirected=True, max_iterations=200)
P.run(st, g)
deg = g.out_degrees()
dmax = int(deg.max())
rng = np.random.default_rng(7)
for b in (100, 1000, 10000, 100000):
    e = rng.integers(0, n, size=(3 * b, 2))
    e = e[e[:, 0] != e[:, 1]]
    e = np.unique(np.sort(e, axis=1), axis=0)
    e = e[(deg[e[:, 0]] + 1 < dmax) & (deg[e[:, 1]] + 1 < dmax)][:b]
    e = e[~g._present(e)]
    arcs = np.concatenate([e, e[:, ::-1]])
    P.update_batch(st, g, P.EdgeBatch(insertions=[tuple(x) for x in arcs.tolist()]))
    np.add.at(deg, arcs[:, 0], 1)
    dyn = P.ranking_result(st)
    s1 = P.run(P.init(g, crit, undirected=True, max_iterations=200), g)
    s2 = P.run(P.init(g, crit, undirected=True, max_iterations=200), g)
    print(b, "dyn==s1", dyn.top(100) == s1.top(100), "s1==s2", s1.top(100) == s2.top(100),
          "r", dyn.iterations_used, s1.iterations_used, s2.iterations_used,
          "lower eq", bool(np.array_equal(dyn.lower, s1.lower)), bool(np.array_equal(s1.lower, s2.lower)),
          flush=True)
