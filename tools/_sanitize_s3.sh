# compute-sanitizer on the session-3 kernels (late PDL wait, trimmed epilogues) + the cluster split-K variant
mkdir -p gpurun_out
for t in memcheck synccheck racecheck initcheck; do
  echo "== $t"
  timeout 1200 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_run.py > gpurun_out/s3_sanitize_$t.log 2>&1
  echo "rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|ok$" gpurun_out/s3_sanitize_$t.log | head -4
done
for t in memcheck synccheck racecheck; do
  echo "== cluster split-K (IOS_TILE_VARIANT=3) $t"
  IOS_TILE_VARIANT=3 timeout 1200 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_run.py > gpurun_out/s3_sanitize_csk_$t.log 2>&1
  echo "rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|ok$" gpurun_out/s3_sanitize_csk_$t.log | head -4
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 2>&1 | tail -1 | cut -c1-300
