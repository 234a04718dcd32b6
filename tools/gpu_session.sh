mkdir -p gpurun_out
timeout 1200 python bench.py --workload c5 > gpurun_out/g50_c5.log 2>&1; echo "c5 $?"
