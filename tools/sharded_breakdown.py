"""Per-phase host timing of one sharded step (world=1 under torchrun, or any
world): wraps every backend call of ShardedRun with a device sync and a
perf_counter, and times the collectives the same way.

  python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 \
      --master-addr 127.0.0.1 --master-port 29513 tools/sharded_breakdown.py
"""
from __future__ import annotations

import collections
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_03847_b200 as P  # noqa: E402
from paper_1807_03847_b200 import distributed as D  # noqa: E402
from paper_1807_03847_b200 import generators as G  # noqa: E402

SCALE = int(os.environ.get("SCALE", "24"))


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    gfull = G.rmat_graph(1 << SCALE, edge_factor=16, seed=42, device=local)
    ip, ix = gfull.csr_arrays()
    gfull.device_graph.close()
    plan = D.ShardPlan(ip, world)
    crit = P.Criterion.top_k(100, 1e-6)
    d = plan.max_degree
    alpha = 1.0 / (1.0 + d)
    gamma = P.tail_gamma(alpha, d)
    shard = D.CudaShard(plan, rank, ip, ix, device=local, alpha=alpha, gamma=gamma, crit=crit,
                        undirected=True, max_iterations=200)
    shard.collective_device = f"cuda:{local}"
    acc = collections.defaultdict(float)
    cnt = collections.Counter()

    def wrap(obj, name):
        f = getattr(obj, name)

        def g(*a, **k):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out = f(*a, **k)
            torch.cuda.synchronize()
            acc[name] += time.perf_counter() - t0
            cnt[name] += 1
            return out
        setattr(obj, name, g)

    for m in ("iterate", "local_topk", "select_global", "apply_cut", "rank_gathered", "reset",
              "level_tensor", "bounds_tensors"):
        wrap(shard, m)
    real = D._all_gather_flat

    def ag(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        real(*a, **k)
        torch.cuda.synchronize()
        acc["all_gather_flat"] += time.perf_counter() - t0
        cnt["all_gather_flat"] += 1
    D._all_gather_flat = ag

    def step():
        shard.reset(alpha=alpha, gamma=gamma, crit=crit, undirected=True, max_iterations=200)
        return D.ShardedRun(shard, plan, crit, rank=rank, world=world,
                            max_iterations=200).run(host_result=False)

    for _ in range(3):
        step()
    acc.clear()
    cnt.clear()
    reps = 5
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r, _ = step()
    torch.cuda.synchronize()
    tot = (time.perf_counter() - t0) / reps
    if rank == 0:
        print(f"world={world} r={r} step {tot * 1e3:.2f} ms (wrapped, synced)")
        for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
            print(f"  {k:18s} {v / reps * 1e3:8.3f} ms/step  ({cnt[k] // reps} calls)")
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
