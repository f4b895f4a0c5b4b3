set -x
OUT=gpurun_out/rs2
mkdir -p $OUT
B="--no-cpu-baseline --no-e2e --steps 100 --warmup 10"
for rs in 2 1; do
  TAL_RING_SORT=$rs timeout 1200 python bench.py $B --mesh delaunay:2000000 > $OUT/dl_rs${rs}.json 2>> $OUT/err.log
done
TAL_RING_SORT=1 timeout 600 python bench.py $B > $OUT/box_rs1.json 2>> $OUT/err.log
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/rs2/*.json")):
    d = json.load(open(f)); r = d["roofline"]
    print(f, round(d["value"] / 1e9, 2), "Gelem/s  kernel", round(r["kernel_ms"], 4), "step", round(d["ms_per_step"], 4))
PY
