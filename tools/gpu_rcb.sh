set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "loopback" > gpurun_out/pytest_loopback.log 2>&1
for n in 2 3; do
TAL_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n --cells 40 --steps 10 --warmup 3 --check --partition rcb --permute > gpurun_out/bench_dist${n}_rcb.json 2> gpurun_out/bench_dist${n}_rcb.err
done
