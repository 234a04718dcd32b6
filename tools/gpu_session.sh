mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dynamic.py -x -q -k grid > gpurun_out/g91_test.log 2>&1; echo "test $?"
