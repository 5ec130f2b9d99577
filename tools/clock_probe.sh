#!/bin/bash
# sample SM clocks + throttle reasons while a command runs
( for i in $(seq 1 60); do nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv,noheader; sleep 0.25; done ) > gpurun_out/clk.txt &
P=$!
"$@"
kill $P 2>/dev/null
sort gpurun_out/clk.txt | uniq -c | sort -rn | head -8
