rm -f gpurun_out/variants.json
for v in build/var/libtal_noC.so build/var/libtal_pfm3.so paper_2403_08777_b200/libtal_b200.so; do
  for rep in 1 2; do
    TAL_LIB_PATH=$v timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 100 --warmup 10 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'lib':'$v','kernel_ms':d['roofline']['kernel_ms'],'frac':d['roofline']['frac'],'ms_per_step':d['ms_per_step']}))" >> gpurun_out/variants.json 2>>gpurun_out/variants.err
  done
done
