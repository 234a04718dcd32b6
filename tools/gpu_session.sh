mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g9_tests.log 2>&1; echo "tests $?"
