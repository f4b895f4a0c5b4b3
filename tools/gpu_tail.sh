set -x
OUT=gpurun_out/tail
mkdir -p $OUT
B="--no-cpu-baseline --no-e2e --steps 200 --warmup 20"
for rep in 1 2; do
for cp in 128 127 124; do
  timeout 600 python bench.py $B --cta-patches $cp > $OUT/cp${cp}_$rep.json 2>> $OUT/err.log
done
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/tail/*.json")):
    d = json.load(open(f)); r = d["roofline"]
    print(f, round(d["value"] / 1e9, 3), "Gelem/s  kernel", round(r["kernel_ms"], 4), "step", round(d["ms_per_step"], 4), d["prep"]["n_chunks"])
PY
