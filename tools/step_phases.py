"""C2 bench step split into init / run / result, each bracketed by a device
sync and the library timer (kb_timer events on the library stream)."""
from __future__ import annotations

import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_03847_b200 as P  # noqa: E402
from paper_1807_03847_b200 import _lib  # noqa: E402
from paper_1807_03847_b200 import generators as G  # noqa: E402

L = _lib.lib()
g = G.rmat_graph(1 << int(os.environ.get("SCALE", "24")), edge_factor=16, seed=42)
dg = g.device_graph
crit = P.Criterion.top_k(100, 1e-6)
d = g.max_out_degree()
alpha = 1.0 / (1.0 + d)
gamma = P.tail_gamma(alpha, d)
ms = ctypes.c_double()


def timed(fn):
    _lib.check(L.kb_timer(0, 0, None))
    t0 = time.perf_counter()
    out = fn()
    _lib.check(L.kb_timer(0, 1, ctypes.byref(ms)))
    return out, ms.value, 1e3 * (time.perf_counter() - t0)


for rep in range(5):
    h = ctypes.c_void_p()
    _, a, aw = timed(lambda: _lib.check(L.kb_state_create(dg.handle, alpha, gamma, 1, 1, 1e-6,
                                                          100, 0, 0, 1, 200, ctypes.byref(h))))
    conv = ctypes.c_int()
    _, b, bw = timed(lambda: _lib.check(L.kb_run(h, ctypes.byref(conv))))
    pairs = ctypes.c_int64()
    _, c, cw = timed(lambda: _lib.check(L.kb_result(h, None, None, None, ctypes.byref(pairs))))
    print(f"init {a:.3f} ms (wall {aw:.3f}) | run {b:.3f} ms (wall {bw:.3f}) | "
          f"result {c:.3f} ms (wall {cw:.3f}) | total {a + b + c:.3f}", flush=True)
    L.kb_state_destroy(h)
