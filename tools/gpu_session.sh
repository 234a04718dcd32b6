mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_distributed.py -x -q -k device_shard_csr > gpurun_out/g31_tests.log 2>&1; echo "tests $?"
