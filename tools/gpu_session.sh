mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 --sharded --no-cpu --no-e2e > gpurun_out/g89_sh.log 2>&1; echo "sharded $?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 tools/sharded_breakdown.py > gpurun_out/g89_brk.log 2>&1; echo "brk $?"
