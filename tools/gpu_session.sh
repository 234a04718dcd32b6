mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g112_tests.log 2>&1; echo "tests $?"
for b in 0 1; do
  KB_TUNE="result.prefix_bound=$b" timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/g112_c2_b$b.log 2>&1; echo "c2 b=$b $?"
  KB_TUNE="result.prefix_bound=$b" timeout 600 python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/g112_c4_b$b.log 2>&1; echo "c4 b=$b $?"
done
timeout 1500 python bench.py --scale 27 --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/g112_c3.log 2>&1; echo "c3 $?"
