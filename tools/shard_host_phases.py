"""Phases of sharded_run's host-CSR path on one rank (NCCL world 1): the
shard built from the host CSR, the distributed symmetry check, the run."""
import os
import socket
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1807_03847_b200 as P  # noqa: E402
from paper_1807_03847_b200 import _lib  # noqa: E402
from paper_1807_03847_b200 import distributed as D  # noqa: E402
from paper_1807_03847_b200 import generators as G  # noqa: E402

with socket.socket() as so:
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                        device_id=torch.device("cuda", 0))
n = 1 << int(os.environ.get("SCALE", "24"))
g = G.rmat_graph(n, edge_factor=16, seed=42)
ip, ix = (np.ascontiguousarray(a) for a in g.csr_arrays())
L = _lib.lib()
if os.environ.get("PIN", "1") == "1":
    for a in (ip, ix):
        _lib.check(L.kb_host_register(_lib.ptr(a), a.nbytes))
crit = P.Criterion.top_k(100, 1e-6)
d = int(np.diff(ip).max())
plan = D.DevicePlan(n, 1, d)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sh = D.CudaShard(plan, 0, ip, ix, device=0, alpha=1 / (1 + d), gamma=P.tail_gamma(1 / (1 + d), d),
                     crit=crit, undirected=True, max_iterations=200, host_build=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ok = D.shards_symmetric(sh, dist, 1)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    sh.collective_device = "cuda:0"
    res = D.ShardedRun(sh, plan, crit, rank=0, world=1, max_iterations=200).run()
    t3 = time.perf_counter()
    print(f"build {1e3*(t1-t0):.1f} ms, symmetry {1e3*(t2-t1):.1f} ms ({ok}), run+result "
          f"{1e3*(t3-t2):.1f} ms, r={res.iterations_used}", flush=True)
    sh.close()
dist.destroy_process_group()
