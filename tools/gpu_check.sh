# regression check after a change: full GPU suite, smoke, default + 160^3 bench, N>1 paths
set -x
OUT=gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1
timeout 300 python bench.py > $OUT/bench_default.json 2> $OUT/bench.err
timeout 600 python bench.py --cells 160 --steps 100 --warmup 10 > $OUT/bench_160.json 2>> $OUT/bench.err
bash tools/gpu_dist.sh
