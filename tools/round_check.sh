# round-end self check on one GPU: tests, smoke, both bench arms
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/rc_gpu_tests.log 2>&1; echo "gpu tests $?"
timeout 300 python -c 'import __graft_entry__ as g; g.smoke(); print("smoke ok")' > gpurun_out/rc_smoke.log 2>&1; echo "smoke $?"
timeout 900 python bench.py > gpurun_out/rc_bench.log 2>&1; echo "bench $?"
timeout 1800 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/rc_bench_ref.log 2>&1; echo "bench ref $?"
