"""C4 phase split with the library's own device timer: init, run (the
RANKING chain + full checks), result -- each bracketed by kb_timer on the
library stream, after warm-up steps."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_03847_b200 as P  # noqa: E402
from paper_1807_03847_b200 import _lib  # noqa: E402
from paper_1807_03847_b200 import generators as G  # noqa: E402

L = _lib.lib()
g = G.grid_graph(1 << 24)
crit = P.Criterion.ranking(1e-9)
ms = ctypes.c_double()


def timed(f):
    _lib.check(L.kb_timer(0, 0, None))
    t0 = time.perf_counter()
    out = f()
    _lib.check(L.kb_timer(0, 1, ctypes.byref(ms)))
    return out, ms.value, (time.perf_counter() - t0) * 1e3


for rep in range(5):
    st, t_init, w_init = timed(lambda: P.init(g, crit, undirected=True, max_iterations=2000))
    out = ctypes.c_int()
    _, t_run, w_run = timed(lambda: _lib.check(L.kb_run(st._h, ctypes.byref(out))))
    pairs = ctypes.c_int64()
    _, t_res, w_res = timed(lambda: _lib.check(L.kb_result(st._h, None, None, None,
                                                           ctypes.byref(pairs))))
    info = st._info()
    print(f"rep {rep}: init {t_init:.3f} ms, run {t_run:.3f} ms (wall {w_run:.3f}), "
          f"result {t_res:.3f} ms; r={info.r} K1 {info.spmv_ms / max(1, info.spmv_launches):.4f} "
          f"ms x {info.spmv_launches} = {info.spmv_ms:.3f} ms", flush=True)
    del st
