mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -k C5 > gpurun_out/g19_c5.log 2>&1; echo "c5 $?"
