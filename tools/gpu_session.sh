mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_dynamic.py tests/test_gpu_distributed.py -x -q > gpurun_out/g58_tests.log 2>&1; echo "tests $?"
for cw in 0 1; do
  KB_TUNE="k1.combine_warp=$cw" timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/g58_c2_cw$cw.log 2>&1; echo "c2 cw=$cw $?"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_heavy --csv --log-file gpurun_out/g58_hc.csv python tools/k2_one.py > gpurun_out/g58_ncu.log 2>&1; echo "ncu $?"
