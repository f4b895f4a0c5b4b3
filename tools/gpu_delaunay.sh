# Unstructured (Delaunay) mesh: GPU parity tests, a ~13 M-tet bench line with
# parity, and an ncu full set of the private kernel on it
set -x
OUT=gpurun_out/dl
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k delaunay > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
timeout 1200 python bench.py --mesh delaunay:2000000 --steps 100 --warmup 10 --no-e2e > $OUT/bench_delaunay.json 2> $OUT/bench.err
cat $OUT/bench_delaunay.json
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_assemble_private -s 3 -c 1 -o $OUT/prof_delaunay python bench.py --mesh delaunay:2000000 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > $OUT/ncu.log 2>&1
ls -la $OUT
