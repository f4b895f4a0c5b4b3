# code-shape study (B / RS / RSP) on one B200: tests, bench lines, ncu of each shape
set -x
OUT=gpurun_out
timeout 600 python -m pytest tests/test_variants.py -q -m gpu > $OUT/pytest_variants.log 2>&1
for v in b rs; do
  for sc in atomic private; do
    timeout 600 python bench.py --variant $v --scatter $sc --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_shape_${v}_${sc}.json 2>> $OUT/bench_shapes.err
  done
done
timeout 300 python bench.py --scatter atomic --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $OUT/bench_shape_rsp_atomic.json 2>> $OUT/bench_shapes.err
for v in b rs; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_assemble_ -s 3 -c 1 -o $OUT/prof_shape_$v python bench.py --variant $v --scatter atomic --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_shape_$v.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_assemble_atomic -s 3 -c 1 -o $OUT/prof_shape_rsp_atomic python bench.py --scatter atomic --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_shape_rsp.log 2>&1
