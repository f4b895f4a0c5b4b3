set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -q --maxfail=30 > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
rm -f gpurun_out/bench_modes.json
for s in private atomic colored; do timeout 300 python bench.py --scatter $s --no-cpu-baseline --no-e2e --steps 50 --warmup 5 >> gpurun_out/bench_modes.json 2>>gpurun_out/bench.err; done
for r in "--renumber none --element-order keep" "--renumber none --element-order sfc" "--renumber sfc --element-order sfc" "--renumber rcm --element-order node"; do timeout 300 python bench.py $r --no-cpu-baseline --no-e2e --steps 50 --warmup 5 >> gpurun_out/bench_modes.json 2>>gpurun_out/bench.err; done
timeout 300 python bench.py --permute --renumber none --element-order keep --no-cpu-baseline --no-e2e --steps 50 --warmup 5 >> gpurun_out/bench_modes.json 2>>gpurun_out/bench.err
timeout 300 python bench.py --permute --no-cpu-baseline --no-e2e --steps 50 --warmup 5 >> gpurun_out/bench_modes.json 2>>gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_assemble_private -s 3 -c 1 -o gpurun_out/prof_private python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
