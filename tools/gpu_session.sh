mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dynamic.py tests/test_gpu_fullsize.py -x -q > gpurun_out/g85_tests.log 2>&1; echo "tests $?"
for sd in 0 1; do
  KB_TUNE="k1.ovf_side=$sd" EDGES=1000,10000 timeout 900 python tools/c5_trace2.py > gpurun_out/g85_trace_$sd.log 2>&1; echo "trace $sd $?"
done
timeout 1200 python bench.py --workload c5 > gpurun_out/g85_c5.log 2>&1; echo "c5 $?"
