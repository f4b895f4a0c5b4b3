# A/B of environment settings (e.g. VARIANTS="TAL_BANK_PLACE=0 TAL_BANK_PLACE=1") on the in-tree library
rm -f gpurun_out/variants_env.json
for rep in 1 2 3; do
for v in $VARIANTS; do
    env $v timeout 300 python bench.py $BENCH_ARGS --no-cpu-baseline --no-e2e --steps 200 --warmup 20 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'env':'$v','kernel_ms':d['roofline']['kernel_ms'],'frac':d['roofline']['frac'],'ms_per_step':d['ms_per_step'],'parity':(d.get('parity') or {}).get('passed')}))" >> gpurun_out/variants_env.json 2>>gpurun_out/variants.err
done
done
cat gpurun_out/variants_env.json
