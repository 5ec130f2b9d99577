timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 python tools/c2_experiment.py 2>&1 | head -1
timeout 300 python bench.py --config C1 --graph --no-cpu --small-batch 0 --ingest 0 --steps 500 --warmup 20 > gpurun_out/c1g.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/c1g.json')); print('C1 graph', d['ms_per_step']*1e3, 'us')"
timeout 300 python tools/c1_experiment.py 2>&1 | head -2
