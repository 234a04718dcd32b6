mkdir -p gpurun_out
for b in 22 20; do timeout 300 ./tools/micro/tma_gather $b; done > gpurun_out/g90_mix.log 2>&1; echo "mix $?"
