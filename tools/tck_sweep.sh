./tools/pipe_probe
for k in 16 32; do echo "C4 tc_k=$k"; TCK=$k timeout 400 python tools/seed_experiment.py 100000000 4096 2>&1 | tail -1; done
