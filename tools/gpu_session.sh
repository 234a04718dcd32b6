mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g99_tests.log 2>&1; echo "tests $?"
bash tools/checked_suite.sh
for l in 0 1; do
  KB_TUNE="init.lazy=$l" timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/g99_c2_l$l.log 2>&1; echo "c2 l=$l $?"
done
