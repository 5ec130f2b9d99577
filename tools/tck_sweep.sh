# CTA pairs: per-half accumulator handshakes (default) vs whole buffers (tc_debug 1024)
timeout 900 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -2
for d in 0 1024 0 1024; do echo "C4 dbg=$d"; REPS=10 timeout 400 python tools/tc_experiment.py 100000000 $d 2>&1 | tail -1; done
for d in 0 1024; do echo "20M dbg=$d"; REPS=10 timeout 400 python tools/tc_experiment.py 20000000 $d 2>&1 | tail -1; done
