"""C4 (grid 4096^2, ranking 1e-9): step time and K1 ms per tuning variant."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_03847_b200 as P
from paper_1807_03847_b200 import _lib, generators as G
L = _lib.lib()
g = G.grid_graph(1 << 24)
crit = P.Criterion.ranking(1e-9)
grid = json.loads(os.environ.get("GRID", '[{"k1.narrow_q":2},{"k1.narrow_q":4}]'))
for cfg in grid:
    for k, v in cfg.items():
        L.kb_tune(k.encode(), int(v))
    ms = P.engine.ctypes.c_double()
    for rep in range(3):
        st = P.init(g, crit, undirected=True, max_iterations=2000)
        _lib.check(L.kb_timer(0, 0, None))
        out = P.engine.ctypes.c_int()
        _lib.check(L.kb_run(st._h, P.engine.ctypes.byref(out)))
        _lib.check(L.kb_timer(0, 1, P.engine.ctypes.byref(ms)))
        info = st._info()
    print(json.dumps({"cfg": cfg, "run_ms": round(ms.value, 3),
                      "k1_ms": round(info.spmv_ms / max(1, info.spmv_launches), 4), "r": info.r}))
