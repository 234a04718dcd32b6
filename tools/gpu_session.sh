mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g33_tests.log 2>&1; echo "tests $?"
timeout 300 python tools/step_phases.py > gpurun_out/g33_phases.log 2>&1; echo "phases $?"
