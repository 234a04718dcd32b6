mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/g56_tests.log 2>&1; echo "tests $?"
for ec in 0 1; do
  KB_TUNE="k2.early_cut=$ec" timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/g56_c2_ec$ec.log 2>&1; echo "c2 ec=$ec $?"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_topk --csv --log-file gpurun_out/g56_k2.csv python tools/k2_one.py > gpurun_out/g56_ncu.log 2>&1; echo "ncu $?"
