"""C4 step split into init / run / result (host wall time around each call)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_03847_b200 as P
from paper_1807_03847_b200 import _lib, generators as G
L = _lib.lib()
g = G.grid_graph(1 << 24)
crit = P.Criterion.ranking(1e-9)
def step():
    t = [time.perf_counter()]
    st = P.init(g, crit, undirected=True, max_iterations=2000); L.kb_sync(0); t.append(time.perf_counter())
    out = P.engine.ctypes.c_int()
    _lib.check(L.kb_run(st._h, P.engine.ctypes.byref(out))); t.append(time.perf_counter())
    pairs = P.engine.ctypes.c_int64()
    _lib.check(L.kb_result(st._h, None, None, None, P.engine.ctypes.byref(pairs))); t.append(time.perf_counter())
    info = st._info()
    return [round((b - a) * 1e3, 3) for a, b in zip(t, t[1:])] + [round(info.spmv_ms / max(1, info.spmv_launches), 4), info.spmv_launches]
for _ in range(3): step()
for _ in range(3): print("init/run/result ms, k1 ms, k1 launches:", step())
