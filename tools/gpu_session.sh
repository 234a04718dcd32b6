mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_checked_build.py -q > gpurun_out/g17_ck.log 2>&1; echo "ck $?"
bash tools/checked_suite.sh
