# Round-2 multi-rank bench validation on a 1-GPU box (ranks time-share cuda:0,
# host objects over gloo): bench.py self-launches N ranks for --gpus N
set -x
OUT=gpurun_out/r2
mkdir -p $OUT
timeout 600 python bench.py --gpus 2 --scaling strong --cells 64 --check --steps 20 --warmup 3 > $OUT/bench_dist2_strong64.json 2> $OUT/bench_dist2_strong64.err
timeout 600 python bench.py --gpus 3 --scaling weak --cells 48 --check --steps 20 --warmup 3 > $OUT/bench_dist3_weak48.json 2> $OUT/bench_dist3_weak48.err
timeout 600 python bench.py --gpus 2 --scaling strong --cells 64 --check --scatter private --steps 20 --warmup 3 > $OUT/bench_dist2_strong64_exchange.json 2> $OUT/bench_dist2_strong64_exchange.err
timeout 600 python bench.py --gpus 4 --scaling strong --cells 64 --check --partition rcb --permute --steps 10 --warmup 3 > $OUT/bench_dist4_rcb_permuted.json 2> $OUT/bench_dist4_rcb_permuted.err
