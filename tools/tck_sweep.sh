timeout 600 python bench.py > gpurun_out/bench_pw.json 2> gpurun_out/bench_pw.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_pw.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['per_launch']['hbm_gbs'], d['e2e']['value'], d['stages_ms'], d['clocks']); print(d['small_batch']); print(d['mid_batch'])"
