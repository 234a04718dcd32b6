mkdir -p gpurun_out
bash tools/round_check.sh
bash tools/checked_suite.sh
