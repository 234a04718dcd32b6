mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g62_tests.log 2>&1; echo "tests $?"
for f in 1 0; do
  KB_TUNE="chk.pub_host=$f" timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/g62_c2_p$f.log 2>&1; echo "c2 p=$f $?"
  KB_TUNE="chk.pub_host=$f" timeout 600 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/g62_c4_p$f.log 2>&1; echo "c4 p=$f $?"
done
