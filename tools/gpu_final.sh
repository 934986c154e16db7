# final verification pass: sanitizer (incl. lagged scan + litmus), hang watchdogs, GPU suite
mkdir -p gpurun_out
for T in memcheck racecheck synccheck initcheck; do
  echo "== $T" >> gpurun_out/final_sanitize.log
  FORGE_LIB=dev FORGE_SCAN_LAG=16 timeout 1200 compute-sanitizer --tool $T --print-limit 20 python tools/sanitize_run.py >> gpurun_out/final_sanitize.log 2>&1
  echo "rc=$?" >> gpurun_out/final_sanitize.log
done
for op in 12 10 11 0 5 9; do timeout 60 python tools/hang_probe.py $op 600 27 >> gpurun_out/final_hang.log 2>&1; done
for op in 0 11; do timeout 60 python tools/hang_probe.py $op 2000 22 >> gpurun_out/final_hang.log 2>&1; done
timeout 180 python tools/hang_probe2.py 80 28 >> gpurun_out/final_hang.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/final_pytest.log 2>&1; echo rc=$? >> gpurun_out/final_pytest.log
exit 0
