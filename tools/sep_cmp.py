"""kb_result time with the galloping vs the table separated-pair count."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_03847_b200 as P
from paper_1807_03847_b200 import _lib, generators as G
L = _lib.lib()
scale = int(os.environ.get("SCALE", "27"))
g = G.grid_graph(1 << scale) if os.environ.get("GRID") else G.rmat_graph(1 << scale, edge_factor=16, seed=42)
crit = P.Criterion.ranking(1e-9) if os.environ.get("GRID") else P.Criterion.top_k(100, 1e-6)
st = P.init(g, crit, undirected=True, max_iterations=2000)
out = P.engine.ctypes.c_int()
_lib.check(L.kb_run(st._h, P.engine.ctypes.byref(out)))
for tab in (0, 1, 0, 1):
    L.kb_tune(b"result.sep_table", tab)
    pairs = P.engine.ctypes.c_int64()
    L.kb_sync(0); t0 = time.perf_counter()
    _lib.check(L.kb_result(st._h, None, None, None, P.engine.ctypes.byref(pairs)))
    print("table" if tab else "gallop", round((time.perf_counter() - t0) * 1e3, 2), "ms", pairs.value)
