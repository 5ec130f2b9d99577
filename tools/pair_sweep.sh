# CTA pairs vs single CTAs across DB sizes (1,024 frames): where do pairs pay?
for n in 20000000 50000000 100000000; do
  for p in 0 2; do echo "n=$n pair=$p"; PAIR=$p REPS=10 timeout 300 python tools/tc_experiment.py $n 0 2>&1 | tail -1 | cut -c1-100; done
done
