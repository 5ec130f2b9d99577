# graph replay: parity tests, C1 eager vs graph, C5 streaming eager vs graph
timeout 600 python -m pytest tests/test_gpu_graph.py tests/test_gpu_parity.py tests/test_gpu_service.py -x -q > gpurun_out/pytest_graph.log 2>&1; tail -5 gpurun_out/pytest_graph.log
for g in "" "--graph"; do
timeout 300 python bench.py --config C1 --no-cpu --small-batch 0 --ingest 0 --steps 500 --warmup 20 $g > gpurun_out/c1$g.json 2> gpurun_out/c1$g.err; echo rc=$?
python -c "import json,sys; d=json.load(open('gpurun_out/c1$g.json')); print('C1 $g', d['ms_per_step']*1e3, 'us', d['step_ms'], d['e2e'], d.get('graph_replays'))"
timeout 300 python bench.py --config C5 --seconds 3 $g > gpurun_out/c5$g.json 2> gpurun_out/c5$g.err; echo rc=$?
python -c "import json,sys; d=json.load(open('gpurun_out/c5$g.json')); d.pop('config',None); print('C5 $g', json.dumps(d)[:600])"
done
