timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
for g in "" "--graph"; do
timeout 300 python bench.py --config C1 --no-cpu --small-batch 0 --ingest 0 --steps 500 --warmup 20 $g > gpurun_out/c1$g.json 2> gpurun_out/c1$g.err; echo rc=$?
python -c "import json,sys; d=json.load(open('gpurun_out/c1$g.json')); print('C1 $g', d['ms_per_step']*1e3, 'us', d['step_ms'], d['e2e'], d.get('graph_replays'), d['gpu_launches']/d['steps'])"
done
timeout 300 python tools/c1_experiment.py
