mkdir -p gpurun_out
bash tools/round_check.sh
bash tools/checked_suite.sh
timeout 900 python bench.py --workload c4 > gpurun_out/fin_c4.log 2>&1; echo "c4 $?"
timeout 1500 python bench.py --scale 27 > gpurun_out/fin_c3.log 2>&1; echo "c3 $?"
timeout 900 python bench.py --workload c5 > gpurun_out/fin_c5.log 2>&1; echo "c5 $?"
