timeout 600 python -m pytest tests/test_gpu_shift.py -x -q > gpurun_out/pytest_shift.log 2>&1; echo shift=$?
tail -3 gpurun_out/pytest_shift.log
grep -E "Error|assert" gpurun_out/pytest_shift.log | head -5
