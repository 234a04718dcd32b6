mkdir -p gpurun_out
timeout 600 python tools/c4_phases.py > gpurun_out/g84_c4ph.log 2>&1; echo "ph $?"
KB_TUNE="k1.lazy_bounds=1" timeout 600 python tools/c4_phases.py > /dev/null 2>&1
