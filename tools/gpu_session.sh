mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g111_tests.log 2>&1; echo "tests $?"
for p in 0 1; do
  KB_TUNE="result.prefix_sort=$p" timeout 900 python bench.py --steps 10 --warmup 3 --sharded --no-cpu --no-e2e > gpurun_out/g111_sh_p$p.log 2>&1; echo "sharded p=$p $?"
done
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/g111_c2.log 2>&1; echo "c2 $?"
