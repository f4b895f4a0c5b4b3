# GPU test suite + default bench + prep timings at 128^3 / 256^3
set -x
OUT=gpurun_out/r2
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1
tail -3 $OUT/pytest_gpu.log
timeout 400 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
TAL_PREP_TIMES=1 timeout 900 python bench.py --cells 256 --steps 50 --warmup 5 --no-cpu-baseline > $OUT/bench_256.json 2> $OUT/bench_256.err
