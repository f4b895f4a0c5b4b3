# Round-2 evidence on one B200: smoke, GPU tests, every bench line kept under
# profiles/round2/, compute-sanitizer on the new paths.
set -x
OUT=gpurun_out/r2/ev
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1
B="--no-cpu-baseline --no-e2e"
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench.err
timeout 300 python bench.py --scatter private $B > $OUT/bench_private.json 2>> $OUT/bench.err
timeout 300 python bench.py --permute $B > $OUT/bench_permuted_rcm.json 2>> $OUT/bench.err
timeout 300 python bench.py --permute --renumber none --element-order keep $B > $OUT/bench_permuted_none.json 2>> $OUT/bench.err
timeout 300 python bench.py --scatter atomic $B > $OUT/bench_atomic.json 2>> $OUT/bench.err
timeout 300 python bench.py --scatter colored $B > $OUT/bench_colored.json 2>> $OUT/bench.err
timeout 300 python bench.py --scatter sequential $B --steps 20 --warmup 3 > $OUT/bench_sequential.json 2>> $OUT/bench.err
timeout 300 python bench.py --pressure $B > $OUT/bench_pressure.json 2>> $OUT/bench.err
timeout 300 python bench.py --supg $B > $OUT/bench_supg.json 2>> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 10 --warmup 2 > $OUT/bench_reference.json 2>> $OUT/bench.err
timeout 900 python bench.py --cells 160 --steps 100 --warmup 10 $B > $OUT/bench_160cubed.json 2>> $OUT/bench.err
timeout 900 python bench.py --cells 256 --steps 50 --warmup 5 $B > $OUT/bench_256cubed.json 2>> $OUT/bench.err
timeout 600 python bench.py --gpus 2 --scaling strong --cells 64 --check --steps 20 --warmup 3 > $OUT/bench_dist2_strong64.json 2>> $OUT/bench.err
timeout 600 python bench.py --gpus 3 --scaling weak --cells 48 --check --steps 20 --warmup 3 > $OUT/bench_dist3_weak48.json 2>> $OUT/bench.err
timeout 600 python bench.py --gpus 2 --scaling strong --cells 64 --check --scatter private --steps 20 --warmup 3 > $OUT/bench_dist2_strong64_exchange.json 2>> $OUT/bench.err
timeout 600 python bench.py --gpus 4 --scaling strong --cells 64 --check --partition rcb --permute --steps 10 --warmup 3 > $OUT/bench_dist4_rcb_permuted.json 2>> $OUT/bench.err
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py > $OUT/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' $OUT/sanitize_$tool.log | tail -1)" >> $OUT/sanitize_summary.txt
done
ls -la $OUT
