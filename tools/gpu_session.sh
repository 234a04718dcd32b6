mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dynamic.py tests/test_gpu_reference_suite.py -x -q > gpurun_out/g49_tests.log 2>&1; echo "dyn tests $?"
EDGES=10000,100000 timeout 900 python tools/c5_pyprof.py > gpurun_out/g49_pyprof.log 2>&1; echo "prof $?"
