# mbarrier waits: suspend-hint try_wait (default) vs spinning try_wait (1024: MMA warp, 2048: epilogue)
for d in 0 1024 2048 3072 0; do echo "C4 dbg=$d"; REPS=10 timeout 400 python tools/tc_experiment.py 100000000 $d 2>&1 | tail -1; done
