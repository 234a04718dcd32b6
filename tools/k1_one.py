"""Three iterations of the C2 static run (R-MAT s24 ef16): the first K1 is
the gather-free ones step, the next two are k_sell_iterate -- the launch an
ncu capture targets (-k regex:k_sell_iterate -s 1 -c 1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_03847_b200 as P  # noqa: E402
from paper_1807_03847_b200 import generators as G  # noqa: E402

scale = int(os.environ.get("SCALE", "24"))
g = G.rmat_graph(1 << scale, edge_factor=16, seed=42)
st = P.init(g, P.Criterion.top_k(100, 1e-6), undirected=True)
for _ in range(3):
    P.iterate_once(st, g)
print("r =", st.r)
