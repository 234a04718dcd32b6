mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_distributed.py -x -q > gpurun_out/g35_tests.log 2>&1; echo "tests $?"
timeout 900 python tools/shard_host_phases.py > gpurun_out/g36.log 2>&1; echo "phases $?"
timeout 900 python bench.py --steps 5 --warmup 3 --sharded --no-cpu > gpurun_out/g35_sh.log 2>&1; echo "sharded $?"
