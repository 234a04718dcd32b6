mkdir -p gpurun_out
SPLITS='[2048]' GRID='{"k1.cluster":[0,2,4,8],"k1.hot":[12288]}' timeout 900 python tools/k1_sweep.py > gpurun_out/g14_sweep.log 2>&1; echo "sweep $?"
SPLITS='[2048]' GRID='{"k1.cluster":[2,4],"k1.hot":[8192,16384]}' timeout 900 python tools/k1_sweep.py >> gpurun_out/g14_sweep.log 2>&1; echo "sweep2 $?"
