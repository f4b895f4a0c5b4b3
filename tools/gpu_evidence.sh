# Round evidence on one B200: smoke, GPU tests, every bench line kept under profiles/
set -x
OUT=gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1
timeout 300 python bench.py > $OUT/bench_default.json 2> $OUT/bench.err
timeout 300 python bench.py --scatter private --no-cpu-baseline > $OUT/bench_private.json 2>> $OUT/bench.err
timeout 300 python bench.py --permute --no-cpu-baseline --no-e2e > $OUT/bench_permuted_rcm.json 2>> $OUT/bench.err
timeout 300 python bench.py --permute --renumber none --element-order keep --no-cpu-baseline --no-e2e > $OUT/bench_permuted_none.json 2>> $OUT/bench.err
timeout 300 python bench.py --scatter atomic --no-cpu-baseline --no-e2e > $OUT/bench_atomic.json 2>> $OUT/bench.err
timeout 300 python bench.py --scatter colored --no-cpu-baseline --no-e2e > $OUT/bench_colored.json 2>> $OUT/bench.err
timeout 300 python bench.py --scatter sequential --no-cpu-baseline --no-e2e --steps 20 --warmup 3 > $OUT/bench_sequential.json 2>> $OUT/bench.err
timeout 300 python bench.py --pressure --no-cpu-baseline --no-e2e > $OUT/bench_pressure.json 2>> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $OUT/bench_reference.json 2>> $OUT/bench.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 50 --warmup 5 > $OUT/bench_torchrun1.json 2>> $OUT/bench.err
timeout 600 python bench.py --cells 160 --steps 100 --warmup 10 > $OUT/bench_160cubed.json 2>> $OUT/bench.err
timeout 900 python bench.py --cells 256 --steps 50 --warmup 5 > $OUT/bench_256cubed.json 2>> $OUT/bench.err
