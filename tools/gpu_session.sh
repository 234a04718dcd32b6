mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_dynamic.py -x -q > gpurun_out/g16_tests.log 2>&1; echo "tests $?"
timeout 300 python tools/step_phases.py > gpurun_out/g16_phases.log 2>&1; echo "phases $?"
