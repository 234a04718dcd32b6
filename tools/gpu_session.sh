mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_sep --csv --log-file gpurun_out/g66_c2.csv python tools/k2_one.py > gpurun_out/g66_ncu.log 2>&1; echo "ncu $?"
SCALE=27 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_sep --csv --log-file gpurun_out/g66_c3.csv python tools/k2_one.py > gpurun_out/g66_ncu3.log 2>&1; echo "ncu $?"
