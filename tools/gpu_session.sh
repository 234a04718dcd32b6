# scratch driver for one gpurun call (edited per experiment); default: the
# round-end self check plus the checked-build suite
mkdir -p gpurun_out
bash tools/round_check.sh
bash tools/checked_suite.sh
