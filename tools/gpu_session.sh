mkdir -p gpurun_out
timeout 900 python tools/k3_runs.py > gpurun_out/g51_k3runs.log 2>&1; echo "k3 $?"
