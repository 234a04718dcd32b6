mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k device_loop > gpurun_out/g28_tests.log 2>&1; echo "tests $?"
