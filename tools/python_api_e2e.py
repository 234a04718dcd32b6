"""The reference-style Python path at C2, end to end: host CSR in a Graph,
init (upload + ingest), run, and the RankingResult arrays read back into
numpy (pageable memory throughout)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1807_03847_b200 as P
from paper_1807_03847_b200 import generators as G
dg = G.rmat_graph(1 << int(os.environ.get("SCALE", "24")), edge_factor=16, seed=42)
ip, ix = (np.ascontiguousarray(a) for a in dg.csr_arrays())
dg.device_graph.close()
crit = P.Criterion.top_k(100, 1e-6)
for rep in range(4):
    g = P.Graph.from_csr(ip.size - 1, ip, ix)
    t0 = time.perf_counter()
    st = P.init(g, crit, undirected=True)
    t1 = time.perf_counter()
    res = P.run(st, g)
    t2 = time.perf_counter()
    o, lo, up = np.asarray(res.order), np.asarray(res.lower), np.asarray(res.upper)
    t3 = time.perf_counter()
    print(f"init(upload+ingest) {1e3*(t1-t0):.1f} ms, run {1e3*(t2-t1):.1f} ms, "
          f"read order/lower/upper {1e3*(t3-t2):.1f} ms, total {1e3*(t3-t0):.1f} ms")
    del st, res
