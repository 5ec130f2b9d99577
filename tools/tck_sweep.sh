# seed sample count (new CTA-per-job select) vs seed time, survivors, scan at C4
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "seed or tau" 2>&1 | tail -2
timeout 600 python tools/seed_experiment.py 100000000 4096,8192,16384,32768,4096 2>&1 | tail -5
