mkdir -p gpurun_out
for R in 1 5 9 13 17 29 28; do
  echo "ring=$R" >> gpurun_out/ring3.log
  FORGE_LIB=dev FORGE_SCAN_RING=$R timeout 300 python tools/probe.py scan >> gpurun_out/ring3.log 2>&1
done
