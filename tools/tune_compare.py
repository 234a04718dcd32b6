"""Time C2 (or C4 with WORKLOAD=c4) K1 with a knob on/off: KNOB=name VALUES=0,1"""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_03847_b200 as P
from paper_1807_03847_b200 import _lib, generators as G

L = _lib.lib()
knob = os.environ.get("KNOB", "k1.narrow4").encode()
vals = [int(v) for v in os.environ.get("VALUES", "0,1").split(",")]
wl = os.environ.get("WORKLOAD", "c2")
if wl == "c4":
    g = G.grid_graph(1 << 24)
    crit = P.Criterion.ranking(1e-9)
else:
    g = G.rmat_graph(1 << int(os.environ.get("SCALE", "24")), edge_factor=16, seed=42)
    crit = P.Criterion.top_k(100, 1e-6)
for rep in range(2):
    for v in vals:
        L.kb_tune(knob, v)
        st = P.init(g, crit, undirected=True, max_iterations=2000)
        t0 = time.perf_counter()
        res = P.run(st, g)
        dt = time.perf_counter() - t0
        lo = res.lower
        import hashlib
        dig = hashlib.sha256(np.ascontiguousarray(lo).tobytes()).hexdigest()[:16]
        i = st._info()
        print(json.dumps({"knob": knob.decode(), "value": v, "rep": rep, "run_s": round(dt, 5),
                          "k1_ms": round(i.spmv_ms / max(1, i.spmv_launches), 4), "r": i.r,
                          "top3": res.top(3), "lower_sha": dig}), flush=True)
