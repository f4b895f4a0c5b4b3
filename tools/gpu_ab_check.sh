# A/B of build/var/*.so vs the in-tree library (interleaved timing reps) plus
# the GPU parity test file run against every variant library
rm -f gpurun_out/variants.json gpurun_out/variants_parity.log
for v in build/var/*.so; do
  echo "== $v" >> gpurun_out/variants_parity.log
  TAL_LIB_PATH=$v timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2 >> gpurun_out/variants_parity.log
done
for rep in 1 2 3; do
for v in build/var/*.so paper_2403_08777_b200/libtal_b200.so; do
    TAL_LIB_PATH=$v timeout 300 python bench.py $BENCH_ARGS --no-cpu-baseline --no-e2e --steps 200 --warmup 20 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'lib':'$v','kernel_ms':d['roofline']['kernel_ms'],'frac':d['roofline']['frac'],'ms_per_step':d['ms_per_step']}))" >> gpurun_out/variants.json 2>>gpurun_out/variants.err
done
done
cat gpurun_out/variants_parity.log
