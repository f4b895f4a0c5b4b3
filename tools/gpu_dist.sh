# N>1 code paths on a single-GPU box: ranks time-share cuda:0; host objects over
# gloo.  fused = kernel REDs into the neighbour's RHS via CUDA IPC (default for
# private-atomic); exchange = NCCL-style send/recv path (staged via host under gloo)
set -x
for n in 2 3; do
TAL_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n bench.py --gpus $n --cells 48 --steps 10 --warmup 3 --check > gpurun_out/bench_dist$n.json 2> gpurun_out/bench_dist$n.err
TAL_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n --cells 48 --steps 10 --warmup 3 --check --scatter private > gpurun_out/bench_dist${n}_x.json 2> gpurun_out/bench_dist${n}_x.err
done
