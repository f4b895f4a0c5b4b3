# single-GPU rate vs mesh size (Kuhn boxes 32^3 .. 256^3)
set -x
OUT=gpurun_out/sizes
mkdir -p $OUT
for c in 32 48 64 96 128 160 192 224 256; do
  timeout 900 python bench.py --cells $c --no-cpu-baseline --no-e2e --steps 100 --warmup 10 > $OUT/c$c.json 2>> $OUT/err.log
done
python - <<'PY'
import json
for c in (32, 48, 64, 96, 128, 160, 192, 224, 256):
    d = json.load(open(f"gpurun_out/sizes/c{c}.json")); r = d["roofline"]
    print(c, d["config"]["n_elems"], round(d["value"]/1e9, 2), "Gelem/s step", round(d["ms_per_step"], 4), "kernel", round(r["kernel_ms"], 4), "frac", round(r["frac"], 3), round(r["frac_of_nominal"], 3), "prep", round(d["prep"]["native_prep_seconds"], 2))
PY
