for r in 1 2; do for c in 1 2 4 8; do CLUSTER=$c timeout 300 python tools/seed_experiment.py 100000000 4096; done; done
for c in 1 2 8; do CLUSTER=$c timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:tcscan_kernel --launch-skip 3 -c 1 python tools/seed_experiment.py 100000000 4096 2>&1 | grep -E "dram__bytes|gpu__time"; done
