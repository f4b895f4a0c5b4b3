# N>1 code path on a single-GPU box: ranks time-share cuda:0, interface planes
# exchanged with gloo through host memory (validation only; numbers meaningless)
set -x
for n in 2 3; do
TAL_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n bench.py --gpus $n --cells 48 --steps 10 --warmup 3 --check > gpurun_out/bench_dist$n.json 2> gpurun_out/bench_dist$n.err
done
