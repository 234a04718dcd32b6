mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/g71_tests.log 2>&1; echo "tests $?"
for f in 0 1; do
  KB_TUNE="chk.finish_narrow=$f" timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/g71_c2_f$f.log 2>&1; echo "c2 f=$f $?"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_topk_finish --csv --log-file gpurun_out/g71_fin.csv python tools/k2_one.py > gpurun_out/g71_ncu.log 2>&1; echo "ncu $?"
