mkdir -p gpurun_out
SPLITS='[2048]' GRID='{"k1.xload":[0,3,4],"k1.warm":[0,20000,32768,65536,131072],"k1.hot":[12288]}' timeout 900 python tools/k1_sweep.py > gpurun_out/g12_sweep.log 2>&1; echo "sweep $?"
SPLITS='[2048]' GRID='{"k1.xload":[3],"k1.warm":[32768],"k1.hot":[8192,16384,20480]}' timeout 900 python tools/k1_sweep.py >> gpurun_out/g12_sweep.log 2>&1; echo "sweep2 $?"
