for n in 100000000 20000000; do echo "n=$n"; REPS=10 timeout 400 python tools/tc_experiment.py $n 0 2>&1 | tail -1; done
