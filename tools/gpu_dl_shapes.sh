set -x
OUT=gpurun_out/dls
mkdir -p $OUT
B="--no-cpu-baseline --no-e2e --steps 100 --warmup 10 --mesh delaunay:2000000"
for cp in 128 256 64; do
  timeout 1200 python bench.py $B --cta-patches $cp --chunk-nodes $((cp * 2)) > $OUT/dl_cp$cp.json 2>> $OUT/err.log
done
timeout 1200 python bench.py $B --renumber sfc > $OUT/dl_sfc.json 2>> $OUT/err.log
timeout 1200 python bench.py $B --element-order node > $OUT/dl_eonode.json 2>> $OUT/err.log
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/dls/*.json")):
    try:
        d = json.load(open(f)); r = d["roofline"]
        print(f, round(d["value"] / 1e9, 2), "Gelem/s  kernel", round(r["kernel_ms"], 4), d["prep"]["n_chunks"])
    except Exception as e:
        print(f, "failed", e)
PY
