mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dynamic.py -x -q > gpurun_out/g48_tests.log 2>&1; echo "dyn tests $?"
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q -k "C5" > gpurun_out/g48_c5.log 2>&1; echo "c5 tests $?"
EDGES=100,1000,10000,100000 timeout 900 python tools/c5_trace2.py > gpurun_out/g48_trace.log 2>&1; echo "trace $?"
