"""cProfile of init on a host Graph at C2 (pageable arrays)."""
import cProfile, io, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1807_03847_b200 as P
from paper_1807_03847_b200 import generators as G
dg = G.rmat_graph(1 << 24, edge_factor=16, seed=42)
ip, ix = (np.ascontiguousarray(a) for a in dg.csr_arrays())
dg.device_graph.close()
crit = P.Criterion.top_k(100, 1e-6)
for rep in range(2):
    g = P.Graph.from_csr(ip.size - 1, ip, ix)
    pr = cProfile.Profile(); pr.enable()
    st = P.init(g, crit, undirected=True)
    pr.disable()
    del st
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(14); print(s.getvalue()[-3000:])
