"""kb_graph_create from page-locked vs pageable host arrays at C2."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1807_03847_b200 as P
from paper_1807_03847_b200 import _lib, generators as G
L = _lib.lib()
g = G.rmat_graph(1 << 24, edge_factor=16, seed=42)
ip, ix = (np.ascontiguousarray(a) for a in g.csr_arrays())
def t_create(reps=3):
    out = []
    for _ in range(reps):
        t0 = time.perf_counter(); dg = P.DeviceGraph(ip, ix); out.append(time.perf_counter() - t0); dg.close()
    return [round(x * 1e3, 1) for x in out]
print("pageable", t_create())
for a in (ip, ix): L.kb_host_register(_lib.ptr(a), a.nbytes)
print("pinned", t_create())
for a in (ip, ix): L.kb_host_unregister(_lib.ptr(a))
for rep in range(3):
    t0 = time.perf_counter()
    for a in (ip, ix): L.kb_host_register(_lib.ptr(a), a.nbytes)
    t1 = time.perf_counter()
    dg = P.DeviceGraph(ip, ix); t2 = time.perf_counter(); dg.close()
    for a in (ip, ix): L.kb_host_unregister(_lib.ptr(a))
    t3 = time.perf_counter()
    print("register %.1f create %.1f unregister %.1f ms" % ((t1-t0)*1e3, (t2-t1)*1e3, (t3-t2)*1e3))
