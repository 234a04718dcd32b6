"""cProfile of one sharded e2e step (world 1) on C2."""
import cProfile, io, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29581")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
import numpy as np, torch, torch.distributed as dist
import paper_1807_03847_b200 as P
from paper_1807_03847_b200 import _lib, distributed as D, generators as G
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
L = _lib.lib()
n = 1 << 24
g = G.rmat_graph(n, edge_factor=16, seed=42)
ip, ix = g.csr_arrays()
plan = D.ShardPlan(ip, 1)
crit = P.Criterion.top_k(100, 1e-6)
alpha = 1.0 / (1.0 + plan.max_degree); gamma = P.tail_gamma(alpha, plan.max_degree)
lcsr = tuple(np.ascontiguousarray(x) for x in plan.local_csr(ip, ix, 0))
out = (np.empty(n, dtype=np.int64), np.empty(n), np.empty(n))
for a in lcsr + out:
    L.kb_host_register(_lib.ptr(a), a.nbytes)
def step():
    sh = D.CudaShard(plan, 0, None, None, device=0, alpha=alpha, gamma=gamma, crit=crit,
                     undirected=True, max_iterations=200, split_threshold=D.fast_split(1),
                     local_csr=lcsr)
    sh.collective_device = "cuda:0"
    t1 = time.perf_counter()
    r = D.ShardedRun(sh, plan, crit, rank=0, world=1, max_iterations=200).run(True, out=out)
    t2 = time.perf_counter()
    sh.close()
    return t1, t2
step(); step()
t0 = time.perf_counter(); pr = cProfile.Profile(); pr.enable(); t1, t2 = step(); pr.disable(); t3 = time.perf_counter()
print(f"create {1e3*(t1-t0):.1f} ms, run+result {1e3*(t2-t1):.1f} ms, close {1e3*(t3-t2):.1f}")
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(12); print(s.getvalue()[-2600:])
dist.destroy_process_group()
