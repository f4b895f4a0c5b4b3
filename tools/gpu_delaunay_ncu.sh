set -x
OUT=gpurun_out/dl3
mkdir -p $OUT
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_assemble_private -s 3 -c 1 -o $OUT/prof_delaunay_final python bench.py --mesh delaunay:2000000 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > $OUT/ncu.log 2>&1
ls -la $OUT
