mkdir -p gpurun_out
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/g29_smoke.log 2>&1; echo "smoke $?"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dynamic.py -x -q > gpurun_out/g29_tests.log 2>&1; echo "tests $?"
