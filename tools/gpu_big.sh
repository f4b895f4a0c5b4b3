# larger configs on one B200 (256^3 = configs[3] total size, 160^3 = configs[4]
# per-GPU slab), e2e slots A/B, and register/occupancy variants A/B
set -x
OUT=gpurun_out
timeout 900 python bench.py --cells 256 --steps 50 --warmup 5 > $OUT/bench_256.json 2> $OUT/bench_big.err
timeout 600 python bench.py --cells 160 --steps 100 --warmup 10 > $OUT/bench_160.json 2>> $OUT/bench_big.err
for rep in 1 2; do
  timeout 300 python bench.py --no-cpu-baseline --steps 50 --warmup 5 > $OUT/bench_slots3_$rep.json 2>> $OUT/bench_big.err
  TAL_LIB_PATH=build/var/libtal_slots4.so timeout 300 python bench.py --no-cpu-baseline --steps 50 --warmup 5 > $OUT/bench_slots4_$rep.json 2>> $OUT/bench_big.err
done
rm -f $OUT/variants.json
for v in build/var/libtal_m3.so build/var/libtal_u2.so build/var/libtal_u2m3.so build/var/libtal_u3m3.so paper_2403_08777_b200/libtal_b200.so; do
  for rep in 1 2; do
    TAL_LIB_PATH=$v timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 100 --warmup 10 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'lib':'$v','kernel_ms':d['roofline']['kernel_ms'],'frac':d['roofline']['frac'],'ms_per_step':d['ms_per_step']}))" >> $OUT/variants.json 2>>$OUT/variants.err
  done
done
