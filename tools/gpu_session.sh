mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/g44_tests.log 2>&1; echo "tests $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g44_smoke.log 2>&1; echo "smoke $?"
