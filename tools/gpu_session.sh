mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/g25_b.log 2>&1; echo "b $?"
