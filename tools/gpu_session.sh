mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dynamic.py -x -q -k "respread or overflow" > gpurun_out/g70_tests.log 2>&1; echo "tests $?"
