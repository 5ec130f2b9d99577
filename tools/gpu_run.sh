CMD="python tools/tc_experiment.py 100000000 0"
timeout 300 $CMD > gpurun_out/exp_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tcscan -s 3 -c 1 -o gpurun_out/prof_tc3 $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
tail -2 gpurun_out/exp_plain.log
