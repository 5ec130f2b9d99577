set -x
python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m "gpu" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --small-batch 0"
timeout 900 $CMD > gpurun_out/b_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 3 -c 1 -o gpurun_out/prof_scan $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench=$?
tail -2 gpurun_out/bench.log
