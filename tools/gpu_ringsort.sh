# A/B of the within-chunk ring-length sort (TAL_RING_SORT) on the Kuhn box
# (128^3) and an unstructured Delaunay mesh (2 M points, 13.5 M tets), plus
# the GPU test suite with the sort on (the default)
set -x
OUT=gpurun_out/rs
mkdir -p $OUT
B="--no-cpu-baseline --no-e2e --steps 100 --warmup 10"
for rep in 1 2; do
  for rs in 0 1; do
    TAL_RING_SORT=$rs timeout 600 python bench.py $B > $OUT/box_rs${rs}_$rep.json 2>> $OUT/err.log
  done
done
for rs in 0 1; do
  TAL_RING_SORT=$rs timeout 1200 python bench.py $B --mesh delaunay:2000000 > $OUT/dl_rs${rs}.json 2>> $OUT/err.log
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/rs/*.json")):
    d = json.load(open(f)); r = d["roofline"]
    print(f, round(d["value"] / 1e9, 2), "Gelem/s  kernel", round(r["kernel_ms"], 4), "step", round(d["ms_per_step"], 4))
PY
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; tail -2 $OUT/pytest_gpu.log
