# Round-2 final evidence on one B200: everything in gpu_r2_evidence.sh plus
# the multi-rank validation lines (ranks time-sharing cuda:0)
bash tools/gpu_r2_evidence.sh
OUT=gpurun_out/r2/ev
timeout 600 python bench.py --gpus 2 --scaling strong --cells 128 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/bench_dist2_strong128.json 2>> $OUT/bench.err
timeout 900 python bench.py --gpus 2 --scaling weak --cells 160 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/bench_dist2_weak160.json 2>> $OUT/bench.err
ls -la $OUT
timeout 1200 python bench.py --mesh delaunay:2000000 --steps 100 --warmup 10 --no-e2e > $OUT/bench_delaunay.json 2>> $OUT/bench.err
