mkdir -p gpurun_out
bash tools/round_check.sh
bash tools/checked_suite.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/fin_ncu.log 2>&1; echo "ncu $?"
