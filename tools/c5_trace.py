"""C5 phase probe: host-side cProfile + device phase trace (KB_TRACE=1) of
update_batch for one insertion batch on R-MAT s24 ef16."""
import cProfile, io, os, pstats, sys, time
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
for b in [int(x) for x in os.environ.get("BATCHES", "100,1000,10000,100000").split(",")]:
    e = rng.integers(0, n, size=(3 * b, 2))
    e = e[e[:, 0] != e[:, 1]]
    e = np.unique(np.sort(e, axis=1), axis=0)
    e = e[(deg[e[:, 0]] + 1 < dmax) & (deg[e[:, 1]] + 1 < dmax)][:b]
    e = e[~g._present(e)]
    arcs = np.concatenate([e, e[:, ::-1]])
    batch = P.EdgeBatch(insertions=[tuple(x) for x in arcs.tolist()])
    print(f"=== batch {b}", file=sys.stderr, flush=True)
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    P.update_batch(st, g, batch)
    pr.disable()
    t1 = time.perf_counter() - t0
    np.add.at(deg, arcs[:, 0], 1)
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(14)
    print(f"batch {b}: {t1 * 1e3:.1f} ms", flush=True)
    print(s.getvalue(), flush=True)
