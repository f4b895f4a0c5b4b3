# ncu evidence for the default bench configuration (one GPU)
set -x
OUT=gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/ncu_launch_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_assemble_private -s 3 -c 1 -o $OUT/prof_default python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_assemble_private -s 3 -c 1 -o $OUT/prof_ordered python bench.py --scatter private --steps 4 --warmup 3 --no-cpu-baseline --no-e2e >> $OUT/ncu_full.log 2>&1
