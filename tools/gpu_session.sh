mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_dynamic.py -x -q > gpurun_out/g96_tests.log 2>&1; echo "tests $?"
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/g96_c2.log 2>&1; echo "c2 $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_heavy_combine --csv --log-file gpurun_out/g96_hc.csv python tools/k2_one.py > gpurun_out/g96_ncu.log 2>&1; echo "ncu $?"
