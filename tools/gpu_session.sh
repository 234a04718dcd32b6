mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g21_tests.log 2>&1; echo "tests $?"
timeout 300 python tools/step_phases.py > gpurun_out/g21_phases.log 2>&1; echo "phases $?"
