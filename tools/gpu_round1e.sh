set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -q --maxfail=30 > gpurun_out/pytest_gpu.log 2>&1
rm -f gpurun_out/bench_modes.json
for cfg in "--cta-patches 128 --chunk-nodes 256" "--cta-patches 64 --chunk-nodes 144"; do
 for s in private-atomic private; do
  timeout 300 python bench.py $cfg --scatter $s --no-cpu-baseline --no-e2e --steps 100 --warmup 10 >> gpurun_out/bench_modes.json 2>>gpurun_out/bench.err
 done
done
timeout 300 python bench.py --permute --no-cpu-baseline --no-e2e --steps 50 --warmup 5 >> gpurun_out/bench_modes.json 2>>gpurun_out/bench.err
timeout 300 python bench.py --permute --renumber none --element-order keep --no-cpu-baseline --no-e2e --steps 50 --warmup 5 >> gpurun_out/bench_modes.json 2>>gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_assemble_private -s 3 -c 1 -o gpurun_out/prof_star64 python bench.py --cta-patches 64 --chunk-nodes 144 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
