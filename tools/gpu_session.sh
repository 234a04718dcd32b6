mkdir -p gpurun_out
for pf in 2 24 34 44; do
  KB_TUNE="k1.narrow_pf=$pf" timeout 600 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/g55_c4_pf$pf.log 2>&1; echo "c4 pf=$pf $?"
done
KB_TUNE="k1.narrow_pf=24" timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k C4 > gpurun_out/g55_c4_test.log 2>&1; echo "c4 test $?"
