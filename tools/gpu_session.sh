mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/g109_tests.log 2>&1; echo "tests $?"
for p in 0 1; do
  KB_TUNE="result.prefix_sort=$p" timeout 1500 python bench.py --scale 27 --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/g109_c3_p$p.log 2>&1; echo "c3 p=$p $?"
  KB_TUNE="result.prefix_sort=$p" timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/g109_c2_p$p.log 2>&1; echo "c2 p=$p $?"
done
