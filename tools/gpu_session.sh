mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dynamic.py tests/test_gpu_fullsize.py -x -q > gpurun_out/g88_tests.log 2>&1; echo "tests $?"
for d in 0 1; do
  KB_TUNE="dyn.k1_diff=$d" timeout 1200 python bench.py --workload c5 > gpurun_out/g88_c5_d$d.log 2>&1; echo "c5 d=$d $?"
done
