mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k prefix > gpurun_out/g106_test.log 2>&1; echo "test $?"
