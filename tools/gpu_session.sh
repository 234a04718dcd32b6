mkdir -p gpurun_out
python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/g24_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_rs_downsweep -s 2 -c 1 -o gpurun_out/r02_rs_down python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/g24_ncu.log 2>&1; echo "ncu $?"
