set -x
timeout 700 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
timeout 500 python bench.py > gpurun_out/bench_k32.json 2> gpurun_out/bench_k32.err; tail -c 300 gpurun_out/bench_k32.err
bash tools/ncu_tc.sh
