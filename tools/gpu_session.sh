mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g63_tests.log 2>&1; echo "tests $?"
for b in 0 1; do
  KB_TUNE="result.bucket_sort=$b" timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/g63_c2_b$b.log 2>&1; echo "c2 b=$b $?"
done
KB_TUNE="result.bucket_sort=1" timeout 600 python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/g63_c4.log 2>&1; echo "c4 $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g63_c2.csv python tools/k2_one.py > gpurun_out/g63_ncu.log 2>&1; echo "ncu $?"
