mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_distributed.py tests/test_gpu_parity.py -x -q > gpurun_out/g5_tests.log 2>&1; echo "tests $?"
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/g5_c2.log 2>&1; echo "c2 $?"
timeout 900 python bench.py --steps 5 --warmup 3 --scale 27 > gpurun_out/g5_c3.log 2>&1; echo "c3 $?"
timeout 900 python bench.py --steps 5 --warmup 3 --sharded --no-cpu > gpurun_out/g5_sh.log 2>&1; echo "sharded $?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/g5_ref.log 2>&1; echo "ref $?"
