"""Host-side time of one C2 bench step (init / run / result) around the device work."""
import cProfile, io, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_03847_b200 as P
from paper_1807_03847_b200 import _lib, generators as G
L = _lib.lib()
g = G.rmat_graph(1 << int(os.environ.get("SCALE", "24")), edge_factor=16, seed=42)
crit = P.Criterion.top_k(100, 1e-6)
def step():
    t = [time.perf_counter()]
    st = P.init(g, crit, undirected=True, max_iterations=200); L.kb_sync(0); t.append(time.perf_counter())
    out = P.engine.ctypes.c_int()
    _lib.check(L.kb_run(st._h, P.engine.ctypes.byref(out))); t.append(time.perf_counter())
    pairs = P.engine.ctypes.c_int64()
    _lib.check(L.kb_result(st._h, None, None, None, P.engine.ctypes.byref(pairs))); t.append(time.perf_counter())
    return [round((b - a) * 1e3, 3) for a, b in zip(t, t[1:])]
for _ in range(3): step()
print("init/run/result ms:", [step() for _ in range(3)])
pr = cProfile.Profile(); pr.enable(); step(); pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(8); print(s.getvalue()[-1800:])
