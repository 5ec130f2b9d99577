set -x
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo tc=$?
tail -30 gpurun_out/pytest_tc.log
