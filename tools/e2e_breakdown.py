"""Time the pieces of the e2e path on C2: H2D+ingest, symmetry, init, run, result D2H."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1807_03847_b200 as P
from paper_1807_03847_b200 import _lib, generators as G

L = _lib.lib()
g = G.rmat_graph(1 << 24, edge_factor=16, seed=42)
ip, ix = g.csr_arrays()
ip, ix = np.ascontiguousarray(ip), np.ascontiguousarray(ix)
L.kb_host_register(_lib.ptr(ip), ip.nbytes)
L.kb_host_register(_lib.ptr(ix), ix.nbytes)
crit = P.Criterion.top_k(100, 1e-6)
import torch
for rep in range(int(os.environ.get("REPS", "3"))):
    free, total = torch.cuda.mem_get_info(0)
    print(f"rep {rep}: device free {free/2**30:.1f} GiB of {total/2**30:.1f}", flush=True)
    t = [time.perf_counter()]
    dg = P.DeviceGraph(ip, ix); t.append(time.perf_counter())
    hg = G.DeviceResidentGraph(dg); t.append(time.perf_counter())
    sym = hg.is_symmetric(); t.append(time.perf_counter())
    md = hg.max_out_degree(); t.append(time.perf_counter())
    st = P.init(hg, crit, undirected=True); t.append(time.perf_counter())
    res = P.run(st, hg); t.append(time.perf_counter())
    names = ["create(H2D+ingest)", "wrap", "is_symmetric", "max_degree", "init", "run+result(D2H)"]
    print({n: round(t[i + 1] - t[i], 4) for i, n in enumerate(names)}, flush=True)
    del st, res
    dg.close()
