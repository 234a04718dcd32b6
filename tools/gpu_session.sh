mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_distributed.py -x -q > gpurun_out/g34_tests.log 2>&1; echo "tests $?"
