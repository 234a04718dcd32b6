# scratch driver for one gpurun call (edited per experiment); default: the
# round-end self check plus the checked-build suite
mkdir -p gpurun_out
bash tools/round_check.sh
bash tools/checked_suite.sh
timeout 1500 python bench.py --scale 27 > gpurun_out/fin4_c3.log 2>&1; echo "c3 $?"
timeout 900 python bench.py --workload c4 > gpurun_out/fin4_c4.log 2>&1; echo "c4 $?"
timeout 900 python bench.py --workload c5 > gpurun_out/fin4_c5.log 2>&1; echo "c5 $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin4_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/fin4_ncu.log 2>&1; echo "ncu $?"
