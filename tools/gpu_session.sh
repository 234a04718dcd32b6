mkdir -p gpurun_out
timeout 600 python tools/step_phases.py > gpurun_out/g110_phases.log 2>&1; echo "ph $?"
