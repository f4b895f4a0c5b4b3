set -x
OUT=gpurun_out/ncusrc
mkdir -p $OUT
K="ncu --set full --clock-control none --import-source on -k regex:k_assemble_private -s 3 -c 1"
S="--steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-graph"
timeout 900 $K -o $OUT/prof_default python bench.py $S > $OUT/ncu.log 2>&1
ls -la $OUT
