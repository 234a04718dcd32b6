mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g113_tests.log 2>&1; echo "tests $?"
for i in 1 2; do timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/g113_c2_$i.log 2>&1; echo "c2 $?"; done
