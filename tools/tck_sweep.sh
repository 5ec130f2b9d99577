# exact warps' idle back-off cap: 1024 ns (default) vs 128 ns (tc_debug 2048)
for n in 100000000 20000000 1000000; do for d in 0 2048 0 2048; do echo "n=$n dbg=$d"; REPS=10 timeout 400 python tools/tc_experiment.py $n $d 2>&1 | tail -1; done; done
