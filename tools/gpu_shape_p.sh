set -x
OUT=gpurun_out
timeout 600 python -m pytest tests/test_variants.py -q -m gpu > $OUT/pytest_variants.log 2>&1
timeout 600 python bench.py --variant p --scatter atomic --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_shape_p_atomic.json 2> $OUT/bench_shapes.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_assemble_baseline -s 3 -c 1 -o $OUT/prof_shape_p python bench.py --variant p --scatter atomic --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_shape_p.log 2>&1
