mkdir -p gpurun_out
timeout 1500 python bench.py --scale 27 > gpurun_out/fin3_c3.log 2>&1; echo "c3 $?"
timeout 900 python bench.py > gpurun_out/fin3_c2.log 2>&1; echo "c2 $?"
