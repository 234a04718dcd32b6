"""Where K1's cold gathers come from at C2: arcs by row-degree class, the
share whose column lies outside the shared-memory hot set, and how many
(row, column-block) segments a column-blocked heavy-row pass would make."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1807_03847_b200 import generators as G

scale = int(os.environ.get("SCALE", "24"))
g = G.rmat_graph(1 << scale, edge_factor=16, seed=42)
ip, ix = g.csr_arrays()
n = ip.size - 1
deg = np.diff(ip)
order = np.lexsort((np.arange(n), -deg))      # new id -> original id
newid = np.empty(n, dtype=np.int64)
newid[order] = np.arange(n)
HOT = 12288
cnew = newid[ix]
cold = cnew >= HOT
rdeg = np.repeat(deg, deg)
nnz = ix.size
print(f"n={n} nnz={nnz} nv={(deg > 0).sum()} cold={cold.sum() / nnz:.3f}")
for T in (128, 256, 512, 1024, 2048):
    heavy = rdeg > T
    rows = (deg > T).sum()
    print(f"deg>{T:5d}: rows {rows:8d} arcs {heavy.sum() / nnz:.3f} "
          f"cold arcs in them {(heavy & cold).sum() / nnz:.3f} of nnz "
          f"({(heavy & cold).sum() / cold.sum():.3f} of cold)")
nv = int((deg > 0).sum())
for B in (16384, 24576):
    for T in (512, 2048):
        heavy = rdeg > T
        src = np.repeat(np.arange(n), deg)[heavy]
        blk = cnew[heavy] // B
        pairs = np.unique(src * ((nv + B - 1) // B + 1) + blk).size
        print(f"block {B} deg>{T}: blocks {(nv + B - 1) // B} segments {pairs} "
              f"arcs/segment {heavy.sum() / pairs:.1f}")
