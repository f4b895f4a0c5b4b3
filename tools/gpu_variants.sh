# A/B timing of build variants (build/var/*.so) on the default bench config,
# reps interleaved across variants (same box, same clocks)
OUT=${VAR_OUT:-gpurun_out/r2}
mkdir -p $OUT
rm -f $OUT/variants.json
for rep in 1 2 3; do
  for v in build/var/*.so; do
    TAL_LIB_PATH=$v timeout 300 python bench.py $BENCH_ARGS --no-cpu-baseline --no-e2e --steps 100 --warmup 10 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'lib':'$v','kernel_ms':d['roofline']['kernel_ms'],'frac':d['roofline']['frac'],'ms_per_step':d['ms_per_step'],'parity':(d.get('parity') or {}).get('passed')}))" >> $OUT/variants.json 2>>$OUT/variants.err
  done
done
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open(__import__("os").environ.get("VAR_OUT","gpurun_out/r2")+"/variants.json"):
    r = json.loads(l); d[r["lib"]].append(r["kernel_ms"])
for k, v in d.items():
    print(f"{k:30s} kernel ms {min(v):.4f} (reps {', '.join('%.4f' % x for x in v)})")
PY
