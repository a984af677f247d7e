mkdir -p gpurun_out
for t in memcheck synccheck racecheck initcheck; do
  echo "== $t"
  timeout 1200 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_run.py > gpurun_out/r2_sanitize_$t.log 2>&1
  echo "rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|ok$|Error|error" gpurun_out/r2_sanitize_$t.log | head -12
done
