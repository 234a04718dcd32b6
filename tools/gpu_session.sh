mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k level1 > gpurun_out/g94_test.log 2>&1; echo "test $?"
