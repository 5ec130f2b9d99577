#!/bin/bash
# ncu captures for the round's profiles: (1) --set full of one tcscan_kernel launch at
# C4 (1,024 frames x 100M rows), (2) the per-launch list of one bench step.
set -x
mkdir -p gpurun_out
REPS=1 CHUNK=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:tcscan_kernel \
  --launch-skip 1 -c 1 -o gpurun_out/prof_tc_r01final -f python tools/tc_experiment.py 100000000 0 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --small-batch 0 \
  > gpurun_out/ncu_launches.log 2>&1
tail -n 3 gpurun_out/ncu_full.log; tail -n 3 gpurun_out/ncu_launches.log
