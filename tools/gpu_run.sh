timeout 1500 python -m pytest tests -m "gpu" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python tools/sb_experiment.py 100000000 8
