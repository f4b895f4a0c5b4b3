# Seam check on one B200: the seam GPU tests, then the default bench line
# (its seam_in_reference_driver leg times the reference's own driver at 1
# and 16 threads around the fast seam)
set -x
OUT=gpurun_out/r2s
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "seam or elements" > $OUT/pytest_seam.log 2>&1
tail -3 $OUT/pytest_seam.log
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_default.json 2> $OUT/bench_default.err
python -c "import json; d=json.load(open('$OUT/bench_default.json')); print(json.dumps(d['seam_in_reference_driver'], indent=1)); print(d['roofline']['kernel_ms'], d['e2e'])"
