"""A few iterations of the C4 run (grid 4096^2, ranking 1e-9) -- the launches
an ncu capture targets (-k regex:k_sell_narrow -s 2 -c 1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_03847_b200 as P  # noqa: E402
from paper_1807_03847_b200 import generators as G  # noqa: E402

g = G.grid_graph(1 << 24)
st = P.init(g, P.Criterion.ranking(1e-9), undirected=True, max_iterations=200)
res = P.run(st, g)
print("r =", st.r)
