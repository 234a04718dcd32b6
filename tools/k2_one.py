"""One C2 static run (R-MAT s24 ef16, top-100): the TOPK checks an ncu
capture targets (-k regex:k_topk_select; the first check's select is launch
0, the second check's full select launch 2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_03847_b200 as P  # noqa: E402
from paper_1807_03847_b200 import generators as G  # noqa: E402

g = G.rmat_graph(1 << int(os.environ.get("SCALE", "24")), edge_factor=16, seed=42)
st = P.init(g, P.Criterion.top_k(100, 1e-6), undirected=True)
res = P.run(st, g)
print("r =", st.r, res.top(5))
