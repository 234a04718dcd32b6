mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g4_tests.log 2>&1; echo "tests $?"
timeout 300 python tools/step_phases.py > gpurun_out/g4_phases.log 2>&1; echo "phases $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/g4_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/g4_ncu.log 2>&1; echo "ncu $?"
