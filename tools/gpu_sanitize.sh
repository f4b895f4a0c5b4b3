OUT=gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py > $OUT/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> $OUT/sanitize_summary.txt
done
