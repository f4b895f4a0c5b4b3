# small meshes: 64- vs 128-patch CTAs
set -x
OUT=gpurun_out/small
mkdir -p $OUT
for c in 32 48 64 96; do
  for cp in 128 64; do
    cn=$([ $cp = 64 ] && echo 144 || echo 256)
    timeout 600 python bench.py --cells $c --cta-patches $cp --chunk-nodes $cn --no-cpu-baseline --no-e2e --steps 200 --warmup 20 > $OUT/c${c}_cp$cp.json 2>> $OUT/err.log
  done
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/small/*.json")):
    d = json.load(open(f)); r = d["roofline"]
    print(f, round(d["value"]/1e9, 2), "Gelem/s step", round(d["ms_per_step"], 4), "kernel", round(r["kernel_ms"], 4), d["prep"]["n_chunks"])
PY
