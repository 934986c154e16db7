mkdir -p gpurun_out
for L in 384 448 512 576 640 768; do
  echo "lag=$L" >> gpurun_out/lag2.log
  FORGE_LIB=dev FORGE_SCAN_LAG=$L timeout 300 python tools/probe.py scan >> gpurun_out/lag2.log 2>&1
done
FORGE_LIB=dev FORGE_SCAN_LAG=512 timeout 1200 python -m pytest tests -m gpu -q -x -k "scan or stress or group or semantics" -p no:randomly > gpurun_out/pytest_lag.log 2>&1; echo rc=$? >> gpurun_out/pytest_lag.log
timeout 1200 python -m pytest tests -m gpu -q -x -k "scan or stress or group or semantics" -p no:randomly > gpurun_out/pytest_nolag.log 2>&1; echo rc=$? >> gpurun_out/pytest_nolag.log
