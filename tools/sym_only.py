import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_1807_03847_b200 as P
from paper_1807_03847_b200 import _lib, generators as G
L = _lib.lib()
g = G.rmat_graph(1 << 24, edge_factor=16, seed=42)
ip, ix = g.csr_arrays()
g.device_graph.close()
dg = P.DeviceGraph(ip, ix)
t=time.perf_counter(); s=dg.is_symmetric(); print('sym', s, time.perf_counter()-t)
