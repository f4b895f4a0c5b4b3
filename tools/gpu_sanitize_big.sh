OUT=gpurun_out
for tool in racecheck memcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py big > $OUT/sanitize_big_$tool.log 2>&1
  echo "$tool rc=$?" >> $OUT/sanitize_summary.txt
done
