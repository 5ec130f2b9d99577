# one --set full capture of C1's scan2_kernel and tau_seed_kernel (graph off, eager)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"scan2_kernel|tau_seed_kernel|aggregate_kernel" -c 3 -o gpurun_out/c1_full python bench.py --config C1 --no-cpu --no-e2e --small-batch 0 --ingest 0 --steps 3 --warmup 3 > gpurun_out/ncu_c1.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/c1_full.ncu-rep --page details --csv > gpurun_out/c1_full_details.csv 2>&1; echo rc=$?
