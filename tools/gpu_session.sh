mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g73_tests.log 2>&1; echo "tests $?"
for pf in 2 9; do
  KB_TUNE="k1.lazy_bounds=0,k1.narrow_pf=$pf" timeout 600 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/g73_c4nl_pf$pf.log 2>&1; echo "c4 nl pf=$pf $?"
done
timeout 600 python bench.py --workload c4 --steps 10 --warmup 3 > gpurun_out/g73_c4.log 2>&1; echo "c4 $?"
