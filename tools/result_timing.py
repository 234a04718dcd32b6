"""Device time of kb_run and kb_result (no host outputs) on C2, per knob value."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_03847_b200 as P
from paper_1807_03847_b200 import _lib, generators as G

L = _lib.lib()
knob = os.environ.get("KNOB", "k3.split_sort").encode()
vals = [int(v) for v in os.environ.get("VALUES", "0,1").split(",")]
g = G.rmat_graph(1 << int(os.environ.get("SCALE", "24")), edge_factor=16, seed=42)
crit = P.Criterion.top_k(100, 1e-6)
ms = ctypes.c_double()
for rep in range(3):
    for v in vals:
        L.kb_tune(knob, v)
        st = P.init(g, crit, undirected=True, max_iterations=200)
        out = ctypes.c_int()
        L.kb_timer(0, 0, None)
        _lib.check(L.kb_run(st._h, ctypes.byref(out)))
        L.kb_timer(0, 1, ctypes.byref(ms))
        t_run = ms.value
        pairs = ctypes.c_int64()
        L.kb_timer(0, 0, None)
        _lib.check(L.kb_result(st._h, None, None, None, ctypes.byref(pairs)))
        L.kb_timer(0, 1, ctypes.byref(ms))
        print(json.dumps({"knob": knob.decode(), "value": v, "rep": rep, "run_ms": round(t_run, 3),
                          "result_ms": round(ms.value, 3), "pairs": pairs.value}), flush=True)
