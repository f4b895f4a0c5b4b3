BENCH_ARGS="--scatter private" bash tools/gpu_ab.sh
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "private or merge or bitwise or mid or 32" > gpurun_out/pytest_parity.log 2>&1
