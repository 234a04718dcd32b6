mkdir -p gpurun_out
for b in 24 23 22 20; do timeout 300 ./tools/micro/tma_stream_gather $b; done > gpurun_out/g76_micro.log 2>&1; echo "micro $?"
