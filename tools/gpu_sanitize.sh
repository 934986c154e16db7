mkdir -p gpurun_out
for T in memcheck racecheck synccheck initcheck; do
  echo "== $T" >> gpurun_out/sanitize.log
  FORGE_LIB=dev FORGE_SCAN_LAG=16 timeout 1200 compute-sanitizer --tool $T --print-limit 20 python tools/sanitize_run.py >> gpurun_out/sanitize.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize.log
done
exit 0
