set -x
OUT=gpurun_out/cap
mkdir -p $OUT
B="--no-cpu-baseline --no-e2e --steps 100 --warmup 10 --mesh delaunay:2000000"
for cap in 8 6 5 4; do
  TAL_MAX_RING_TETS=$cap timeout 1200 python bench.py $B > $OUT/dl_cap$cap.json 2>> $OUT/err.log
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/cap/*.json")):
    d = json.load(open(f)); r = d["roofline"]
    print(f, round(d["value"]/1e9, 2), "Gelem/s kernel", round(r["kernel_ms"], 4), d["prep"]["n_patches"], d["prep"]["n_chunks"], d["parity"] and d["parity"]["passed"])
PY
