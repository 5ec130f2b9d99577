timeout 300 python tools/c1_experiment.py
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c1_graph_launches.csv python bench.py --config C1 --graph --no-cpu --no-e2e --small-batch 0 --ingest 0 --steps 5 --warmup 3 > /dev/null 2>&1; echo ncu rc=$?
