# A/B: build/var/*.so against the in-tree library (interleaved reps), then GPU tests on the in-tree library
rm -f gpurun_out/variants.json
for rep in 1 2 3; do
for v in build/var/*.so paper_2403_08777_b200/libtal_b200.so; do
    TAL_LIB_PATH=$v timeout 300 python bench.py $BENCH_ARGS --no-cpu-baseline --no-e2e --steps 200 --warmup 20 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'lib':'$v','kernel_ms':d['roofline']['kernel_ms'],'frac':d['roofline']['frac'],'ms_per_step':d['ms_per_step'],'parity':(d.get('parity') or {}).get('passed')}))" >> gpurun_out/variants.json 2>>gpurun_out/variants.err
done
done
if [ -z "$NO_TESTS" ]; then timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log; fi
cat gpurun_out/variants.json
