mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/g100_c2.log 2>&1; echo "c2 $?"
timeout 900 python bench.py --workload c5 > gpurun_out/g100_c5.log 2>&1; echo "c5 $?"
timeout 900 python bench.py --workload c4 > gpurun_out/g100_c4.log 2>&1; echo "c4 $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g100_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/g100_ncu.log 2>&1; echo "ncu $?"
