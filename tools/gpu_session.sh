mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k own_radix > gpurun_out/g30_tests.log 2>&1; echo "tests $?"
KB_TUNE=result.own_sort=1 timeout 300 python tools/step_phases.py > gpurun_out/g30_phases.log 2>&1; echo "phases $?"
KB_TUNE=result.own_sort=1 timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/g30_plain.log 2>&1 && KB_TUNE=result.own_sort=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/g30_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/g30_ncu.log 2>&1; echo "ncu $?"
