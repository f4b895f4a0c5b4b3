# Round-2 ncu evidence: launch list of the default bench, ncu --set full of
# the dominant kernel for config 2 (private-atomic, private) and config 3
# (random node permutation, with and without RCM renumbering), with the bench
# line of the same configuration next to each; plus the FP64 probe table.
set -x
OUT=gpurun_out/r2/ncu
mkdir -p $OUT
./tools/probe_fp64 > $OUT/probe_fp64.txt 2>&1
B="--no-cpu-baseline --no-e2e --steps 30 --warmup 5"
timeout 300 python bench.py $B > $OUT/bench_default.json 2>/dev/null
timeout 300 python bench.py $B --permute --renumber none --element-order keep > $OUT/bench_permuted_none.json 2>/dev/null
timeout 300 python bench.py $B --permute > $OUT/bench_permuted_rcm.json 2>/dev/null
timeout 300 python bench.py $B --scatter private > $OUT/bench_private.json 2>/dev/null
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/ncu_launch_bench.log 2>&1
K="ncu --set full --clock-control none --import-source on -k regex:k_assemble_private -s 3 -c 1"
S="--steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-graph"
timeout 600 $K -o $OUT/prof_default python bench.py $S > $OUT/ncu_full.log 2>&1
timeout 600 $K -o $OUT/prof_private python bench.py $S --scatter private >> $OUT/ncu_full.log 2>&1
timeout 600 $K -o $OUT/prof_permuted_none python bench.py $S --permute --renumber none --element-order keep >> $OUT/ncu_full.log 2>&1
timeout 600 $K -o $OUT/prof_permuted_rcm python bench.py $S --permute >> $OUT/ncu_full.log 2>&1
ls -la $OUT
