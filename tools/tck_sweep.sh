# threshold refresh period: every 4 own tiles (default), 2 (tc_debug 2048), 8 (1024)
for n in 100000000 20000000 1000000; do for d in 2048 3072; do echo "n=$n dbg=$d"; REPS=10 timeout 400 python tools/tc_experiment.py $n $d 2>&1 | tail -1; done; done
