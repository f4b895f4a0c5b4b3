# Round-2 single-GPU bench lines + the reference arm (numba reference on the host)
set -x
OUT=gpurun_out/r2
mkdir -p $OUT
timeout 400 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout 600 python bench.py --impl reference --steps 10 --warmup 2 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
