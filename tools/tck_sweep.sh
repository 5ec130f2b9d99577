# survivor-row L2 prefetch at enqueue (default) vs none (tc_debug 512)
for n in 100000000 20000000 1000000; do for d in 0 512 0 512; do echo "n=$n dbg=$d"; REPS=10 timeout 400 python tools/tc_experiment.py $n $d 2>&1 | tail -1; done; done
