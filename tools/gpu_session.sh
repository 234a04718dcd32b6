mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_distributed.py tests/test_gpu_dynamic.py -x -q > gpurun_out/g18_tests.log 2>&1; echo "tests $?"
timeout 900 python bench.py --workload c4 > gpurun_out/g18_c4.log 2>&1; echo "c4 $?"
