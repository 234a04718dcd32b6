mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dynamic.py tests/test_gpu_fullsize.py -k "C5 or dynamic or update or batch or heavy or golden" -x -q > gpurun_out/g26_tests.log 2>&1; echo "tests $?"
timeout 900 python tools/c5_trace2.py > gpurun_out/g26_c5.log 2>&1; echo "c5 $?"
